import numpy as np, sys
sys.path.insert(0, '/root/repo')
from paper_1603_08109_b200 import gpa_filter, make_spatial_kernel, synth
from oracle import gpa_oracle as orc
for (H, Wd) in ((2100, 2100), (1990, 2100)):
    img = np.floor(synth.config_image("c4", height=H, width=Wd)).astype(np.float32)
    for W, N in ((1, 7), (5, 8), (20, 57)):
        k = make_spatial_kernel("box", half_width=W)
        o32 = gpa_filter(img, k, 25.0, N, precision="f32")
        o64 = gpa_filter(img, k, 25.0, N, precision="f64")
        d = np.abs(o32 - o64)
        j = np.unravel_index(int(np.argmax(d)), d.shape)
        y, x = j
        sub = img[max(0,y-3):y+4, max(0,x-3):x+4]
        ref = orc.gpa(img[max(0,y-20):y+21, max(0,x-20):x+21].astype(np.float64), "box", W, k.weights_1d, 25.0, N)
        yy, xx = y - max(0, y-20), x - max(0, x-20)
        print(H, Wd, W, N, "max", d.max(), "at", j, "val", img[j], "o32", o32[j], "o64", o64[j], "oracle", ref[yy, xx], "n>1e-4", int((d>1e-4).sum()))
        print(sub)
