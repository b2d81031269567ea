"""Build a variant of libfbgpu.so with extra nvcc -D flags into abtest/<name>.so (A/B timing).

  python tools/ab_build.py NAME -DFB_K2_BOX_MINB=2
  gpurun -- python tools/prof_driver.py --config c4 --lib abtest/NAME.so
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402

name, extra = sys.argv[1], tuple(sys.argv[2:])
g.compile_library(os.path.join(ROOT, "abtest", name + ".so"), os.path.join(ROOT, "abtest", name + "_obj"), extra)
print("built", name)
