"""Build a variant of libfbgpu.so with extra nvcc -D flags into abtest/<name>.so (A/B timing).

  python tools/ab_build.py NAME -DFB_K2_BOX_R=12 -DFB_K2_BOX_WARPS=12
  gpurun -- python tools/prof_driver.py --config c4 --lib abtest/NAME.so
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "abtest", name + "_obj")
os.makedirs(out_dir, exist_ok=True)
procs, objs = [], []
for src in g._sources():
    obj = os.path.join(out_dir, os.path.basename(src).replace(".cu", ".o"))
    procs.append(subprocess.Popen(["nvcc", *g.NVCC_FLAGS, *extra, "-c", "-o", obj, src], cwd=ROOT))
    objs.append(obj)
if any(p.wait() != 0 for p in procs):
    sys.exit("nvcc failed")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                os.path.join(ROOT, "abtest", name + ".so"), *objs], check=True, cwd=ROOT)
print("built", name)
