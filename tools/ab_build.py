"""Build A/B variants of the library with extra -D flags (kernel experiments).

    python tools/ab_build.py name "-DCS_PAIR3_MINB=5" [...]
writes paper_2507_11794_b200/_lib/var_<name>.so; select it at run time with
CLOTHSIM_LIB=<that path>.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11794_b200 import build as B

name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(B.LIB_DIR, f"var_{name}.so")
print(B.build(force=True, extra_flags=flags, out=out))
