"""Build an A/B variant of libbb200.so with extra compile definitions.

    python scripts/build_variant.py OUT.so -DATT_FA_NS=4 [-D...]

Objects go to build_<name>/ next to the package; select the variant at run
time with BB_LIB_PATH=OUT.so (measurement only; the product library is
paper_2605_29233_b200/libbb200.so built by __graft_entry__.build())."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29233_b200 import _build  # noqa: E402

out, defs = os.path.abspath(sys.argv[1]), sys.argv[2:]
name = os.path.splitext(os.path.basename(out))[0]
_build.OBJ = os.path.join(_build.PKG, f"build_{name}")
_build.LIB = out
_build.FLAGS = _build.FLAGS + defs
print(_build.build(force=True))
