"""Build a variant of the library for A/B timing or instrumentation.

  python tools/build_variant.py NAME [-DMACRO ...]   -> build/ab/NAME.so

Same sources and flags as paper_2505_03728_b200/_build.py plus the given
defines; load it with KOP_LIB=build/ab/NAME.so (paper_2505_03728_b200/_lib.py).
ONLY=a.cu,b.cu recompiles just those sources and links the rest from build/obj.
"""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_03728_b200 import _build as b  # noqa: E402


def main():
    name, extra = sys.argv[1], sys.argv[2:]
    out = os.path.join(ROOT, "build", "ab", name)
    os.makedirs(out, exist_ok=True)
    only = [s for s in os.environ.get("ONLY", "").split(",") if s] or b.SOURCES
    jobs = [[b.NVCC, *b.ARCH, *b.FLAGS, *extra, "-c", os.path.join(b.CSRC, s),
             "-o", os.path.join(out, s.replace(".cu", ".o"))] for s in only]
    objs = [os.path.join(out if s in only else b.OBJ, s.replace(".cu", ".o")) for s in b.SOURCES]
    with ThreadPoolExecutor(len(jobs)) as ex:
        for r in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs):
            if r.returncode:
                sys.exit(r.stdout + r.stderr)
    lib = out + ".so"
    subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", lib, *objs, "-lcudart"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
