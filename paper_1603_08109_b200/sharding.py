"""Multi-GPU partitioning (north-star item 5): one process per GPU, no collective on the data path.

Two partitionings:

* by image (`image_shard`): a batch (config c3) is split into contiguous slices of images;
  ranks filter independently.
* by row band (`RowBands`): one huge image (config c4) is split into bands whose first rows
  are multiples of 256 image rows (the box walks of kernel 1 start there, so every rank's
  output is bit-identical to the same rows of a one-GPU call, fbgpu.h `fb_gpa_filter_band`).
  The filter is local with radius W: a rank reads W rows of its neighbours' INPUT bands.
  `PeerInput` maps the neighbours' band buffers over CUDA IPC and hands `fb_gpa_filter_band`
  views of the rows it needs, so kernel 1 reads them in place over NVLink / NVSwitch: no halo
  copy, no extended buffer, no NCCL.  `PeerOutput` is the final gather, fused into kernel 2:
  the root's output buffer is mapped into every rank and each rank's epilogue stores its rows
  straight into it.  The only hand-offs are host-side flags in the job's key-value store
  (`StoreFlags`: "my input band is written", "my rows have landed"), never a device collective
  and never a kernel that waits on another rank's kernel.

`exchange_halos` / `gather_rows` move the same rows with point-to-point messages; they exist
for the CPU (gloo) tests of the partitioning logic, where there is no CUDA IPC.
"""

from __future__ import annotations

from dataclasses import dataclass

#: Row alignment of band starts: every box walk length divides it (fb_common.cuh walk_rows).
BAND_ALIGN = 256


def image_shard(n_images: int, world: int, rank: int) -> range:
    """Contiguous slice of image indices for `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_images, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


@dataclass(frozen=True)
class RowBands:
    """`height` rows split over `world` ranks in units of `align` rows (sizes differ by at most
    one unit; the last band ends at the image's last row)."""

    height: int
    world: int
    W: int
    align: int = BAND_ALIGN

    def __post_init__(self):
        units = -(-self.height // self.align)
        if units < self.world:
            raise ValueError(f"{self.height} rows give fewer than {self.world} bands of {self.align}-row units")

    def bounds(self, rank: int) -> tuple[int, int]:
        units = -(-self.height // self.align)
        base, extra = divmod(units, self.world)
        u0 = rank * base + min(rank, extra)
        u1 = u0 + base + (1 if rank < extra else 0)
        return min(self.height, u0 * self.align), min(self.height, u1 * self.align)

    def halos(self, rank: int) -> tuple[int, int]:
        """(top, bottom) halo rows available from neighbours (0 at the image edges)."""
        r0, r1 = self.bounds(rank)
        return min(self.W, r0), min(self.W, self.height - r1)

    def extended_bounds(self, rank: int) -> tuple[int, int]:
        r0, r1 = self.bounds(rank)
        top, bottom = self.halos(rank)
        return r0 - top, r1 + bottom

    def halo_sources(self, rank: int) -> tuple[tuple[int, int, int] | None, tuple[int, int, int] | None]:
        """Where this rank's halo rows live: (neighbour rank, first row, end row) in that
        neighbour's band coordinates, for the rows above and below (None at an image edge)."""
        top, bottom = self.halos(rank)
        r0, r1 = self.bounds(rank)
        above = below = None
        if top:
            p0, p1 = self.bounds(rank - 1)
            if p1 - p0 < top:
                raise ValueError(f"band of {p1 - p0} rows is thinner than the halo W={self.W}")
            above = (rank - 1, (r0 - top) - p0, r0 - p0)
        if bottom:
            n0, n1 = self.bounds(rank + 1)
            if n1 - n0 < bottom:
                raise ValueError(f"band of {n1 - n0} rows is thinner than the halo W={self.W}")
            below = (rank + 1, 0, bottom)
        return above, below


class StoreFlags:
    """Host-side hand-offs through the job's key-value store (torch.distributed's TCPStore):
    `signal(tag, to)` marks this rank's event `tag` for the ranks `to`; `wait(tag, ranks)` blocks
    until each of `ranks` has signalled it to this rank (a server-side wait, no polling), then
    consumes the flags.  No device collective is involved."""

    def __init__(self, rank: int, store=None):
        import torch.distributed as dist

        self.rank = rank
        self.store = store if store is not None else dist.distributed_c10d._get_default_store()

    def signal(self, tag: str, to) -> None:
        for r in to:
            self.store.set(f"fbgpu/{tag}/{self.rank}>{r}", b"1")

    def wait(self, tag: str, ranks) -> None:
        keys = [f"fbgpu/{tag}/{r}>{self.rank}" for r in ranks]
        if keys:
            self.store.wait(keys)
            for k in keys:
                self.store.delete_key(k)


class PeerInput:
    """The neighbour rows a rank's band needs, read in place from the neighbours' input bands.

    Every rank exports the CUDA IPC handle of its band buffer (setup only: the handles travel
    once through `all_gather_object`); each rank maps its two neighbours' buffers and keeps
    `above` / `below`: `FbImage` views of the W rows next to its band, passed to
    `fb_gpa_filter_band`.  `publish()` / `wait_neighbours()` order a new input against the
    neighbours' reads (a rank re-writing its band must know the neighbours are done with it).
    """

    def __init__(self, band, bands: RowBands, rank: int, device: int, group=None, flags: StoreFlags | None = None):
        import torch
        import torch.distributed as dist

        from . import _native

        self.rank, self.bands = rank, bands
        self.flags = flags or StoreFlags(rank)
        self._gen = 0
        if band.stride(1) != 1:
            raise ValueError("band rows must be contiguous")
        dtype = _native._TORCH_DT[str(band.dtype)]
        itemsize = torch.empty((), dtype=band.dtype).element_size()
        handle, offset = _native.ipc_export(band.data_ptr())
        infos = [None] * bands.world
        dist.all_gather_object(infos, (handle, offset, band.stride(0)), group=group)
        self._bases = []
        self.above = self.below = None
        cols = band.shape[1]
        for which, src in zip(("above", "below"), bands.halo_sources(rank)):
            if src is None:
                continue
            nb, lo, hi = src
            h, off, ld = infos[nb]
            base = _native.ipc_open(device, h)
            self._bases.append(base)
            view = _native.FbImage(base + off + lo * ld * itemsize, dtype, 1, hi - lo, cols, ld)
            setattr(self, which, view)
        self.neighbours = [s[0] for s in bands.halo_sources(rank) if s is not None]

    def publish(self) -> None:
        """This rank's band holds the current input (call after writing it, stream synchronised)."""
        self._gen += 1
        self.flags.signal(f"in{self._gen}", self.neighbours)

    def wait_neighbours(self) -> None:
        """Block until both neighbours published the current input generation."""
        self.flags.wait(f"in{self._gen}", self.neighbours)

    def close(self) -> None:
        from . import _native

        for b in self._bases:
            _native.ipc_close(b)
        self._bases = []


class PeerOutput:
    """The root's full-image output, writable by every rank (north star item 5's final gather,
    fused into the filter's epilogue).

    The root exports the CUDA IPC handle of its output allocation (`fb_ipc_export`); the other
    ranks map it (`fb_ipc_open`) and pass `band(r0, r1)` -- an `FbImage` row slice of the
    root's buffer -- as the output of `_native.gpa_band`.  Kernel 2 then writes those rows over
    NVLink / NVSwitch directly into the root's HBM: no receive buffers, no gather kernel, no
    NCCL call.  `done()` is the hand-off: every filter call is synchronous at return, so a
    rank's rows have landed when it signals; the root waits for every rank's flag.
    """

    def __init__(self, full, shape, dtype, rank: int, device: int, root: int = 0, group=None,
                 flags: StoreFlags | None = None):
        import torch
        import torch.distributed as dist

        from . import _native

        self.rank, self.root, self.group = rank, root, group
        self.world = dist.get_world_size(group)
        self.flags = flags or StoreFlags(rank)
        self._gen = 0
        self.rows, self.cols = shape
        self.dtype = _native._TORCH_DT[str(dtype)]
        self.itemsize = torch.empty((), dtype=dtype).element_size()
        self._base = None
        payload = [None]
        if rank == root:
            if full.stride(1) != 1 or full.stride(0) != self.cols:
                raise ValueError("root buffer must be a contiguous (rows, cols) tensor")
            handle, offset = _native.ipc_export(full.data_ptr())
            payload = [(handle, offset)]
            self.ptr = full.data_ptr()
        dist.broadcast_object_list(payload, src=root, group=group)
        if rank != root:
            handle, offset = payload[0]
            self._base = _native.ipc_open(device, handle)
            self.ptr = self._base + offset

    def band(self, r0: int, r1: int):
        """fb_image for rows [r0, r1) of the root's buffer (device memory of the root GPU)."""
        from . import _native

        return _native.FbImage(self.ptr + r0 * self.cols * self.itemsize, self.dtype, 1, r1 - r0, self.cols,
                               self.cols)

    def done(self) -> None:
        """After this rank's (synchronous) filter call: non-root ranks flag that their rows
        landed; the root returns once every rank has flagged (its buffer is then complete)."""
        self._gen += 1
        tag = f"out{self._gen}"
        if self.rank != self.root:
            self.flags.signal(tag, [self.root])
        else:
            self.flags.wait(tag, [r for r in range(self.world) if r != self.root])

    def close(self):
        from . import _native

        if self._base is not None:
            _native.ipc_close(self._base)
            self._base = None


# ----------------------------------------------------------------------------- CPU (gloo) stand-ins
def exchange_halos(band, W: int, rank: int, world: int, bands: RowBands, group=None):
    """[top halo | band | bottom halo] assembled with point-to-point messages: the rows
    `RowBands.halo_sources` names, moved the way `PeerInput` reads them in place (CPU tests)."""
    import torch
    import torch.distributed as dist

    top, bottom = bands.halos(rank)
    above, below = bands.halo_sources(rank)
    rows, cols = band.shape
    ext = torch.empty((top + rows + bottom, cols), dtype=band.dtype, device=band.device)
    ext[top:top + rows].copy_(band)
    ops = []
    if above is not None:
        ops.append(dist.P2POp(dist.irecv, ext[:top], above[0], group))
    if below is not None:
        ops.append(dist.P2POp(dist.irecv, ext[top + rows:], below[0], group))
    for nb in (rank - 1, rank + 1):  # serve the neighbours' requests for our rows
        if 0 <= nb < world:
            for src in bands.halo_sources(nb):
                if src is not None and src[0] == rank:
                    ops.append(dist.P2POp(dist.isend, band[src[1]:src[2]].contiguous(), nb, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return ext


def gather_rows(out_band, full, rank: int, world: int, bands: RowBands, root: int = 0, group=None):
    """Assemble the full output on `root` from every rank's band (point-to-point into row slices)."""
    import torch.distributed as dist

    if rank == root:
        reqs = []
        for src in range(world):
            r0, r1 = bands.bounds(src)
            if src == root:
                full[r0:r1].copy_(out_band)
            else:
                reqs.append(dist.irecv(full[r0:r1], src, group))
        for req in reqs:
            req.wait()
        return full
    dist.send(out_band.contiguous(), root, group)
    return None

