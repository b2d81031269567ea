import numpy as np

from paper_1603_08109_b200 import synth


def test_synth_deterministic_and_in_range():
    a = synth.synth_image(96, 80, seed=5, n_rects=10, noise_sigma=10.0, smooth_field=True)
    b = synth.synth_image(96, 80, seed=5, n_rects=10, noise_sigma=10.0, smooth_field=True)
    assert a.shape == (96, 80) and a.dtype == np.float32
    assert np.array_equal(a, b)
    assert a.min() >= 0.0 and a.max() <= 255.0


def test_config_shapes():
    c = synth.CONFIGS
    assert (c["c0"].height, c["c0"].dtype) == (512, "float64")
    assert c["c3"].batch == 64 and c["c3"].pixels == 64 * 2048 * 2048
    assert c["c4"].pixels == 16384 * 16384
    img = synth.config_image("c0")
    assert img.shape == (512, 512) and img.dtype == np.float64


def test_golden_crops_regenerate(golden, golden_scalars):
    # The fixtures' inputs are crops of the seeded config images.
    for name in ("c0", "c1"):
        y0, x0 = golden_scalars["cases"][name]["crop_origin"]
        full = synth.config_image(name)
        crop = golden[f"{name}_in"]
        assert np.array_equal(full[y0:y0 + crop.shape[0], x0:x0 + crop.shape[1]], crop)
