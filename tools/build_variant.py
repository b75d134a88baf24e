"""Build an experimental libozk with extra nvcc defines for A/B timing:
python tools/build_variant.py NAME -DFOO=1 ...  ->  tools/_build/libozk_NAME.so
(time it with tools/variants_bench.py; the product build is paper_2301_09960_b200/build.py)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2301_09960_b200 import build as b  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    outdir = os.path.join(ROOT, "tools", "_build")
    os.makedirs(outdir, exist_ok=True)
    out = os.path.join(outdir, f"libozk_{name}.so")

    def compile_one(src):
        obj = os.path.join(outdir, f"{name}.{src}.o")
        subprocess.run([b.NVCC, *b.ARCH, *b.FLAGS, *defs, "-c", os.path.join(b.CSRC, src), "-o",
                        obj], check=True)
        return obj

    def compile_host(src):
        obj = os.path.join(outdir, f"{name}.{src}.o")
        subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-pthread",
                        "-Wno-unknown-pragmas", f"-I{os.path.join(ROOT, 'include')}", "-c",
                        os.path.join(b.CSRC, src), "-o", obj], check=True)
        return obj

    with ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(compile_one, b.SOURCES)) + list(ex.map(compile_host, b.HOST_SOURCES))
    subprocess.run([b.NVCC, *b.ARCH, "-shared", "-cudart", "static", "-ccbin", "g++",
                    "-Xcompiler", "-pthread", "-o", out, *objs], check=True)
    for o in objs:
        os.remove(o)
    print(out)


if __name__ == "__main__":
    main()
