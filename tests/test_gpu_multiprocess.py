"""The multi-GPU data plane run as 2 and 3 processes sharing the one GPU of the test box.

Row bands (config c4's partitioning, sharding.RowBands / PeerInput / PeerOutput): every rank
reads its neighbours' halo rows in place through CUDA IPC mappings of their input bands
(fb_gpa_filter_band) and writes its output rows straight into the root's buffer (the fused
final gather); hand-offs are store flags, no NCCL.  By image (config c3's partitioning): each
rank filters its slice of the batch.  Both must be bit-identical to one process filtering the
whole workload (the box walks start at image rows that are multiples of 256, whatever the split).

IPC needs distinct processes, not distinct devices.  No kernel waits on another rank's kernel:
every filter call is synchronous and the hand-offs are host-side (B200_PROFILING.md).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

H, WD, N_BOX = 2304, 2048, 57  # wpad * H > 4 MP: kernel 1 is the box walker


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)


def _rowband_worker(rank, world, port, out_path, kind):
    import torch
    import torch.distributed as dist

    from paper_1603_08109_b200 import _native, make_spatial_kernel, sharding, synth

    _init(rank, world, port)
    try:
        img = synth.config_image("c4", height=H, width=WD)
        k = make_spatial_kernel("box", half_width=20) if kind == "box" else make_spatial_kernel("gaussian", sigma_s=5.0)
        N = N_BOX if kind == "box" else 42
        bands = sharding.RowBands(H, world, k.half_width)
        r0, r1 = bands.bounds(rank)
        band = torch.from_numpy(np.ascontiguousarray(img[r0:r1])).cuda()
        full = torch.full((H, WD), float("nan"), dtype=torch.float32, device="cuda") if rank == 0 else None
        out = sharding.PeerOutput(full, (H, WD), torch.float32, rank, device=0)
        inp = sharding.PeerInput(band, bands, rank, device=0)
        torch.cuda.synchronize()
        inp.publish()
        inp.wait_neighbours()
        for _ in range(2):  # two steps: the flags of step 1 must not satisfy step 2
            st = _native.gpa_band(band, out.band(r0, r1), k, 25.0, N, 128.0, 128.0, _native.FB_PREC_F32,
                                  row_origin=r0, image_rows=H, above=inp.above, below=inp.below, device=0)
            assert st["h2d_bytes"] == 0 and st["d2h_bytes"] == 0
            out.done()
        if rank == 0:
            np.save(out_path, full.cpu().numpy())
        dist.barrier()  # teardown only: nobody unmaps while a peer still reads
        inp.close()
        out.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["box", "gaussian"])
def test_row_bands_bit_identical_to_single_call(tmp_path, world, kind):
    import torch
    import torch.multiprocessing as mp

    from paper_1603_08109_b200 import _native, make_spatial_kernel, synth

    out_path = str(tmp_path / "full.npy")
    mp.spawn(_rowband_worker, args=(world, _free_port(), out_path, kind), nprocs=world, join=True)
    got = np.load(out_path)
    img = synth.config_image("c4", height=H, width=WD)
    k = make_spatial_kernel("box", half_width=20) if kind == "box" else make_spatial_kernel("gaussian", sigma_s=5.0)
    N = N_BOX if kind == "box" else 42
    ref = torch.empty((H, WD), dtype=torch.float32, device="cuda")
    _native.gpa(torch.from_numpy(img).cuda(), ref, k, 25.0, N, 128.0, 128.0, _native.FB_PREC_F32, 0)
    assert np.array_equal(got, ref.cpu().numpy())


def _batch_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from paper_1603_08109_b200 import gpa_filter_batch, sharding, synth

    _init(rank, world, port)
    try:
        cfg = synth.CONFIGS["c3"]
        idx = list(sharding.image_shard(6, world, rank))
        imgs = [torch.from_numpy(synth.config_image(cfg, i, height=512, width=512)).cuda() for i in idx]
        outs = gpa_filter_batch(imgs, synth.config_kernel(cfg), cfg.sigma_r, 76, precision="f32",
                                out_dtype=np.float32)
        for i, o in zip(idx, outs):
            np.save(os.path.join(out_dir, f"img{i}.npy"), o.cpu().numpy())
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_by_image_shards_bit_identical_to_single_batch(tmp_path, world):
    import torch
    import torch.multiprocessing as mp

    from paper_1603_08109_b200 import gpa_filter_batch, synth

    mp.spawn(_batch_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    cfg = synth.CONFIGS["c3"]
    imgs = [torch.from_numpy(synth.config_image(cfg, i, height=512, width=512)).cuda() for i in range(6)]
    ref = gpa_filter_batch(imgs, synth.config_kernel(cfg), cfg.sigma_r, 76, precision="f32", out_dtype=np.float32)
    for i in range(6):
        assert np.array_equal(np.load(str(tmp_path / f"img{i}.npy")), ref[i].cpu().numpy()), i
