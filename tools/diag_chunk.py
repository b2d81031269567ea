import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_08109_b200 import gpa_filter, synth, make_spatial_kernel
cfg = synth.CONFIGS["c4"]
img = synth.config_image(cfg, height=2304, width=2048)
k = synth.config_kernel(cfg)
N = 57
host = gpa_filter(img, k, 25.0, N, precision="f32")
dev = gpa_filter(torch.from_numpy(img).cuda(), k, 25.0, N, precision="f32").cpu().numpy()
ref = gpa_filter(img, k, 25.0, N, precision="f64")
for name, o in (("host_chunked", host), ("device", dev)):
    d = np.abs(o - ref)
    i = np.unravel_index(np.argmax(d), d.shape)
    print(name, "max", d.max(), "at", i, "p99.99", np.quantile(d, 0.9999), "n>1e-4", int((d > 1e-4).sum()))
d = np.abs(host - dev)
i = np.unravel_index(np.argmax(d), d.shape)
print("host-dev max", d.max(), "at", i, "rows with >1e-4:", sorted(set(np.nonzero(d > 1e-4)[0].tolist()))[:40])
print("img window", img[i[0]-2:i[0]+3, i[1]-2:i[1]+3])
