"""Build experiment variants of libsimplex into build/var_<name>.so (all with the experiment hooks).
    python scripts/var_build.py NAME=DEF[,DEF...] ...      e.g.  RB2=SX_LOOK_RB=2  CB4=SX_LOOK_CB=4
scripts/var_sweep.sh then times each variant (selection phases + pipelined block)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2211_10979_b200 import build  # noqa: E402

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
for spec in sys.argv[1:]:
    name, defs = spec.split("=", 1)
    out = os.path.join(ROOT, "build", f"var_{name}.so")
    build.build(defines=["SIMPLEX_EXPERIMENTS"] + [d for d in defs.split(",") if d], out=out)
    print(out, flush=True)
