"""Multi-GPU partitioning logic on CPU: world_size 2 and 3 over gloo (no GPU needed).

The row-band path takes the W input rows RowBands.halo_sources names from each neighbour
(point-to-point here; PeerInput reads the same rows in place over CUDA IPC on GPUs), filters
its band with them (the CPU oracle stands in for fb_gpa_filter_band), and gathers the bands on
rank 0; the result must equal filtering the whole image.  The store-flag hand-offs that replace
every barrier on the GPU data plane (StoreFlags, PeerOutput.done) run here on gloo's TCPStore.
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
        bands = sharding.RowBands(H, world, W, align=8)
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
    assert bounds == [(2048 * r, 2048 * (r + 1)) for r in range(8)]
    assert b.halos(0) == (0, 20) and b.halos(7) == (20, 0) and b.halos(3) == (20, 20)
    assert b.halo_sources(0) == (None, (1, 0, 20))
    assert b.halo_sources(3) == ((2, 2028, 2048), (4, 0, 20))
    assert b.halo_sources(7) == ((6, 2028, 2048), None)
    for world in (2, 3, 4, 5, 6, 7):  # band starts are multiples of 256 rows (bit-exact bands)
        bw = sharding.RowBands(16384, world, 20)
        bounds = [bw.bounds(r) for r in range(world)]
        assert bounds[0][0] == 0 and bounds[-1][1] == 16384
        assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1))
        assert all(r0 % 256 == 0 for r0, _ in bounds)
        sizes = [r1 - r0 for r0, r1 in bounds]
        assert max(sizes) - min(sizes) <= 256
    ragged = sharding.RowBands(17, 4, 2, align=1)
    assert [ragged.bounds(r) for r in range(4)] == [(0, 5), (5, 9), (9, 13), (13, 17)]
    with pytest.raises(ValueError):
        sharding.RowBands(300, 3, 20)  # two 256-row units cannot make three bands
    with pytest.raises(ValueError, match="thinner"):
        sharding.RowBands(20, 4, 8, align=1).halo_sources(2)


def _flags_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        flags = sharding.StoreFlags(rank)
        log = []
        for step in range(3):
            if rank != 0:
                flags.signal(f"out{step}", [0])
            else:
                flags.wait(f"out{step}", range(1, world))
                log.append(step)
            nbs = [r for r in (rank - 1, rank + 1) if 0 <= r < world]
            flags.signal(f"in{step}", nbs)
            flags.wait(f"in{step}", nbs)
        if rank == 0:
            np.save(out_path, np.array(log))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_store_flag_handoffs(tmp_path, world):
    out_path = str(tmp_path / "log.npy")
    mp.spawn(_flags_worker, args=(world, _free_port(), out_path), nprocs=world, join=True)
    assert np.load(out_path).tolist() == [0, 1, 2]


def test_image_shards_cover_batch():
    for n, world in ((64, 1), (64, 8), (64, 3), (5, 8)):
        shards = [list(sharding.image_shard(n, world, r)) for r in range(world)]
        flat = [i for s in shards for i in s]
        assert flat == list(range(n))
        sizes = [len(s) for s in shards]
        assert max(sizes) - min(sizes) <= 1
