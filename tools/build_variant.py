"""Build an A/B variant of libfj.so with tuning macros, e.g.
   python tools/build_variant.py variants/libfj_i16.so FJ_ITEMS=16
then run any tool with FJ_LIBRARY=<that .so>."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_08143_b200 import build as B  # noqa: E402

out = os.path.abspath(sys.argv[1])
os.makedirs(os.path.dirname(out), exist_ok=True)
print(B.build(force=True, so=out, defines=sys.argv[2:]))
