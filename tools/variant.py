"""Builds a kernel variant of the engine library into tmp_variants/<name>/ with
extra nvcc defines (A/B experiments; select it at run time with HQ_LIB=...).

  python tools/variant.py NAME -DHQ_FOO=1 [-DHQ_BAR=2 ...]
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_16930_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "tmp_variants", name)
    os.makedirs(out, exist_ok=True)
    import glob
    cus = sorted(glob.glob(os.path.join(B.CSRC, "hq_*.cu")))
    flags = [*B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
             "-I", os.path.join(ROOT, "include"), *defs]
    objs = [os.path.join(out, os.path.basename(c)[:-3] + ".o") for c in cus]
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(lambda co: subprocess.check_call([B.NVCC, *flags, "-c", co[0], "-o", co[1]]), zip(cus, objs)))
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", *objs, "-lcublas", "-lcusolver", "-o",
                           os.path.join(out, "libhoqri_b200.so")])
    for o in objs:
        os.remove(o)
    print(os.path.join(out, "libhoqri_b200.so"))


if __name__ == "__main__":
    main()
