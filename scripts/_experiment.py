"""Experiment-only loader (scripts/ probes): build libsimplex with -DSIMPLEX_EXPERIMENTS — the
variant whose SIMPLEX_* environment hooks (SIMPLEX_PROBE, SIMPLEX_PASS_CFG, ...) are live — and
make the binding load it instead of the product libsimplex.so, which never reads the environment.
    import _experiment; _experiment.load()          # before the first Simplex(...)
SIMPLEX_EXPERIMENT_LIB=path selects an already built variant (scripts/var_sweep.sh)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2211_10979_b200 as sx  # noqa: E402
from paper_2211_10979_b200 import build  # noqa: E402

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")


def load(path=None):
    path = path or os.environ.get("SIMPLEX_EXPERIMENT_LIB")
    if not path:
        os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
        path = build.build(defines=["SIMPLEX_EXPERIMENTS"], out=os.path.join(ROOT, "build", "libsimplex_exp.so"))
    sx.use_library(path)
    return path
