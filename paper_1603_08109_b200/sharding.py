"""Multi-GPU partitioning (north-star item 5): one process per GPU over torch.distributed.

Two partitionings, both with no collective on the data path beyond the final gather:

* by image (`image_shard`): a batch (config c3) is split into contiguous
  slices of images; ranks filter independently.
* by row band (`RowBands`): one huge image (config c4) is split into bands of
  H/g rows.  The filter is local with radius W, so each rank needs W rows of
  the INPUT from each neighbour (one point-to-point exchange, 2 x W x cols
  samples, `exchange_halos`) and then filters its band with the halo rows
  passed to the C ABI (`fb_gpa_filter(..., halo_top, halo_bottom, ...)`),
  which replicates only at the true image edges.  The outputs are gathered to
  the root with point-to-point receives into row slices (`gather_rows`).

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
