"""Build a variant of the library for A/B timing or instrumentation.

  python tools/build_variant.py NAME [-DMACRO ...]   -> variants/libkinoptik_b200_NAME.so

Same sources and flags as paper_2505_03728_b200/_build.py plus the given
defines (objects under build/obj_NAME); load it with
KOP_LIB=variants/libkinoptik_b200_NAME.so (paper_2505_03728_b200/_lib.py).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_03728_b200 import _build as b  # noqa: E402

if __name__ == "__main__":
    print(b.build(variant=sys.argv[1], defines=sys.argv[2:]))
