"""A/B experiments: build libbgs.so with extra -D defines into build_variants/<name>/ (the
product build is __graft_entry__.build()); load it with BGS_LIB=<path>.

    python tools/build_variant.py lb32 -DBGS_LOOK_BATCH=32
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
import glob

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "build_variants", name)
    os.makedirs(out, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(ge.CSRC, "*.cu")))

    def comp(src):
        obj = os.path.join(out, os.path.basename(src).replace(".cu", ".o"))
        r = subprocess.run([ge.NVCC, *ge.flags_for(src), *defs, "-c", src, "-o", obj], capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        return obj

    with ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(comp, srcs))
    lib = os.path.join(out, "libbgs.so")
    subprocess.check_call([ge.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs])
    print(lib)


if __name__ == "__main__":
    main()
