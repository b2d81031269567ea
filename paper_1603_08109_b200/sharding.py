"""Multi-GPU partitioning (north-star item 5): one process per GPU over torch.distributed.

Two partitionings, both with no collective on the data path beyond the final gather:

* by image (`image_shard`): a batch (config c3) is split into contiguous
  slices of images; ranks filter independently.
* by row band (`RowBands`): one huge image (config c4) is split into bands of
  H/g rows.  The filter is local with radius W, so each rank needs W rows of
  the INPUT from each neighbour (one point-to-point exchange, 2 x W x cols
  samples, `exchange_halos`) and then filters its band with the halo rows
  passed to the C ABI (`fb_gpa_filter(..., halo_top, halo_bottom, ...)`),
  which replicates only at the true image edges.  The final gather is fused
  into the filter: the root's output buffer is mapped into every rank
  (`PeerOutput`, CUDA IPC over NVLink / NVSwitch) and each rank's kernel 2
  stores its rows straight into it.  `gather_rows` (point-to-point receives
  into row slices) is the same gather as a separate collective, for gloo/CPU.

Over NCCL the point-to-point ops move device memory peer-to-peer over
NVLink/NVSwitch; over gloo the same code runs on CPU tensors (tests).
"""

from __future__ import annotations

from dataclasses import dataclass


def image_shard(n_images: int, world: int, rank: int) -> range:
    """Contiguous slice of image indices for `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_images, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


@dataclass(frozen=True)
class RowBands:
    height: int
    world: int
    W: int

    def bounds(self, rank: int) -> tuple[int, int]:
        base, extra = divmod(self.height, self.world)
        r0 = rank * base + min(rank, extra)
        return r0, r0 + base + (1 if rank < extra else 0)

    def halos(self, rank: int) -> tuple[int, int]:
        """(top, bottom) halo rows available from neighbours (0 at the image edges)."""
        r0, r1 = self.bounds(rank)
        return min(self.W, r0), min(self.W, self.height - r1)

    def extended_bounds(self, rank: int) -> tuple[int, int]:
        r0, r1 = self.bounds(rank)
        top, bottom = self.halos(rank)
        return r0 - top, r1 + bottom


def exchange_halos(band, W: int, rank: int, world: int, bands: RowBands, group=None):
    """Return a tensor [top halo | band | bottom halo] using point-to-point sends/receives.

    `band` is this rank's (rows, cols) tensor.  Rank r sends its first rows to
    rank r-1 (that rank's bottom halo) and its last rows to rank r+1 (that
    rank's top halo).  Bands thinner than W rows are not supported
    (they would need rows from beyond the nearest neighbour).
    """
    import torch
    import torch.distributed as dist

    top, bottom = bands.halos(rank)
    r0, r1 = bands.bounds(rank)
    if world > 1 and (r1 - r0) < W:
        raise ValueError(f"band of {r1 - r0} rows is thinner than the halo W={W}")
    rows, cols = band.shape
    ext = torch.empty((top + rows + bottom, cols), dtype=band.dtype, device=band.device)
    ext[top:top + rows].copy_(band)
    ops = []
    if rank > 0:
        prev_bottom = bands.halos(rank - 1)[1]
        ops.append(dist.P2POp(dist.isend, band[:prev_bottom].contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, ext[:top], rank - 1, group))
    if rank < world - 1:
        next_top = bands.halos(rank + 1)[0]
        ops.append(dist.P2POp(dist.isend, band[rows - next_top:].contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, ext[top + rows:], rank + 1, group))
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


class PeerOutput:
    """The root's full-image output, writable by every rank (north star item 5's final gather,
    fused into the filter's epilogue).

    The root exports the CUDA IPC handle of its output allocation (`fb_ipc_export`); the other
    ranks map it (`fb_ipc_open`) and pass `band(r0, r1)` -- an `FbImage` row slice of the
    root's buffer -- as the output of `_native.gpa`.  Kernel 2 then writes those rows over
    NVLink / NVSwitch directly into the root's HBM: no receive buffers, no gather kernel, no
    NCCL call.  `done()` is the hand-off: each rank's filter call has returned (it synchronises
    its stream), and a barrier tells the root every band has landed.
    """

    def __init__(self, full, shape, dtype, rank: int, device: int, root: int = 0, group=None):
        import torch
        import torch.distributed as dist

        from . import _native

        self.rank, self.root, self.group = rank, root, group
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

    def done(self):
        """Barrier after every rank's (synchronous) filter call: the root's rows are complete."""
        import torch.distributed as dist

        dist.barrier(group=self.group)

    def close(self):
        from . import _native

        if self._base is not None:
            _native.ipc_close(self._base)
            self._base = None
