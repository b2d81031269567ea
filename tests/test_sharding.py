"""Multi-GPU partitioning logic on CPU: world_size 2 over gloo (no GPU needed).

The row-band path exchanges W input rows with each neighbour (point-to-point),
filters its band with the halo rows (here the CPU oracle stands in for
fb_gpa_filter(..., halo_top, halo_bottom)), and gathers the bands on rank 0;
the result must equal filtering the whole image.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import gpa_oracle as orc
from paper_1603_08109_b200 import sharding, synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rowband_worker(rank, world, port, H, Wd, W, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = synth.config_image("c4", height=H, width=Wd).astype(np.float64)
        bands = sharding.RowBands(H, world, W)
        r0, r1 = bands.bounds(rank)
        band = torch.from_numpy(np.ascontiguousarray(img[r0:r1]))
        ext = sharding.exchange_halos(band, W, rank, world, bands)
        top, bottom = bands.halos(rank)
        assert ext.shape[0] == (r1 - r0) + top + bottom
        e0, e1 = bands.extended_bounds(rank)
        assert np.array_equal(ext.numpy(), img[e0:e1])  # halos are the neighbours' real rows
        # stand-in for fb_gpa_filter(ext, halo_top=top, halo_bottom=bottom): filter, keep own rows
        W_, taps, _ = orc.spatial_taps("box", half_width=W)
        out_ext = orc.gpa(ext.numpy(), "box", W_, taps, 25.0, 12)
        out_band = torch.from_numpy(np.ascontiguousarray(out_ext[top:top + (r1 - r0)]))
        full = torch.empty((H, Wd), dtype=torch.float64) if rank == 0 else None
        sharding.gather_rows(out_band, full, rank, world, bands)
        if rank == 0:
            np.save(out_path, full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_bands_with_halo_exchange_match_full_image(tmp_path, world):
    H, Wd, W = 61, 48, 6
    out_path = str(tmp_path / "full.npy")
    mp.spawn(_rowband_worker, args=(world, _free_port(), H, Wd, W, out_path), nprocs=world, join=True)
    img = synth.config_image("c4", height=H, width=Wd).astype(np.float64)
    W_, taps, _ = orc.spatial_taps("box", half_width=W)
    ref = orc.gpa(img, "box", W_, taps, 25.0, 12)
    got = np.load(out_path)
    assert np.max(np.abs(got - ref)) <= 1e-9


def test_band_bounds_and_halos():
    b = sharding.RowBands(16384, 8, 20)
    bounds = [b.bounds(r) for r in range(8)]
    assert bounds[0][0] == 0 and bounds[-1][1] == 16384
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(7))
    assert b.halos(0) == (0, 20) and b.halos(7) == (20, 0) and b.halos(3) == (20, 20)
    ragged = sharding.RowBands(17, 4, 2)
    assert [ragged.bounds(r) for r in range(4)] == [(0, 5), (5, 9), (9, 13), (13, 17)]


def test_image_shards_cover_batch():
    for n, world in ((64, 1), (64, 8), (64, 3), (5, 8)):
        shards = [list(sharding.image_shard(n, world, r)) for r in range(world)]
        flat = [i for s in shards for i in s]
        assert flat == list(range(n))
        sizes = [len(s) for s in shards]
        assert max(sizes) - min(sizes) <= 1
