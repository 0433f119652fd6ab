"""Build kernel variants of libfgtcuda.so (one source recompiled with -D overrides).

    python tools/variants.py k_pw.cu name1:-DFOO=1,-DBAR=2 name2:-DFOO=2
writes build/variants/libfgtcuda_<name>.so; select one at run time with FGT_LIB_PATH.
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_07165_b200 import _build  # noqa: E402


def main():
    src = sys.argv[1]
    _build.build()
    out_dir = os.path.join(ROOT, "build", "variants")
    os.makedirs(out_dir, exist_ok=True)
    nvcc = _build._nvcc()
    objs = [os.path.join(_build.BUILD, s.replace(".cu", ".o")) for s in _build.SOURCES]

    def one(spec):
        name, _, defs = spec.partition(":")
        defs = [d for d in defs.split(",") if d]
        obj = os.path.join(out_dir, f"{src[:-3]}_{name}.o")
        subprocess.run([nvcc] + _build.NVCC_FLAGS + defs + ["-c", os.path.join(_build.CSRC, src), "-o", obj],
                       check=True)
        lib = os.path.join(out_dir, f"libfgtcuda_{name}.so")
        others = [o for o in objs if not o.endswith(src.replace(".cu", ".o"))]
        subprocess.run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib, obj] + others
                       + ["-Xcompiler", "-fPIC"], check=True)
        return lib

    with ThreadPoolExecutor(8) as ex:
        for lib in ex.map(one, sys.argv[2:]):
            print(lib)


if __name__ == "__main__":
    main()
