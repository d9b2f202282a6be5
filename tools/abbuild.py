"""Build variants of libhyena.so with preprocessor switches for A/B measurements on the GPU box:
  python tools/abbuild.py name1:-DX=1,-DY=0 name2:...   -> ab/libhyena_<name>.so
then run bench.py with HYENA_LIB=ab/libhyena_<name>.so (paper_2311_12519_b200/hyena.py)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_12519_b200 import build as b  # noqa: E402


def one(spec):
    name, _, defs = spec.partition(":")
    out = os.path.join(ROOT, "ab", f"libhyena_{name}.so")
    cmd = ["nvcc"] + b.NVCC_FLAGS + [d for d in defs.split(",") if d] + \
          [os.path.join(b.CSRC, s) for s in b.SOURCES] + ["-o", out]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    os.makedirs(os.path.join(ROOT, "ab"), exist_ok=True)
    with ThreadPoolExecutor(len(sys.argv) - 1) as ex:
        for o in ex.map(one, sys.argv[1:]):
            print(o)
