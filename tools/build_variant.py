"""Build a variant of libhhg with extra nvcc defines (development A/B timing).

usage: python tools/build_variant.py NAME [-DMACRO[=V] ...]
-> tools/variants/libhhg_NAME.so; select it with KB_LIB=... in tools/kbench.py
and tools/gsprof.py."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as G  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "tools", "variants")
    od = os.path.join(out, "obj_" + name)
    os.makedirs(od, exist_ok=True)
    srcs = G._sources()

    def cc(src):
        o = os.path.join(od, os.path.basename(src)[:-3] + ".o")
        subprocess.run(["nvcc", *G.NVCC_FLAGS, *defs, "-c", "-o", o, src], check=True, capture_output=True)
        return o

    with ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(cc, srcs))
    so = os.path.join(out, f"libhhg_{name}.so")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", so, *objs,
                    "-Xcompiler", "-fopenmp", "-lgomp", "-lnccl"], check=True)
    print(so)


if __name__ == "__main__":
    main()
