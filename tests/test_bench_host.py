"""bench.py's host-side logic, checked on CPU (the GPU legs run on the box).  bench.py is what the
driver runs at round end, so a NameError in a rarely taken branch (the largest-tableau leg, the
small-tableau roofline) must be caught here, not there: a small static check flags every name a
function reads that no enclosing scope, module global or builtin defines."""
import ast
import builtins
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import lpgen  # noqa: E402


def _bound(node):
    """Names bound directly in a function / lambda / comprehension scope."""
    names = set()
    if isinstance(node, (ast.FunctionDef, ast.AsyncFunctionDef, ast.Lambda)):
        a = node.args
        for x in a.posonlyargs + a.args + a.kwonlyargs:
            names.add(x.arg)
        if a.vararg:
            names.add(a.vararg.arg)
        if a.kwarg:
            names.add(a.kwarg.arg)
    if isinstance(node, (ast.ListComp, ast.SetComp, ast.DictComp, ast.GeneratorExp)):
        stack = [g.target for g in node.generators]
    else:
        stack = list(node.body if isinstance(node.body, list) else [node.body])
    while stack:
        n = stack.pop()
        if isinstance(n, (ast.FunctionDef, ast.AsyncFunctionDef, ast.ClassDef)):
            names.add(n.name)
            continue
        if isinstance(n, (ast.Lambda, ast.ListComp, ast.SetComp, ast.DictComp, ast.GeneratorExp)):
            continue
        if isinstance(n, ast.Name) and isinstance(n.ctx, (ast.Store, ast.Del)):
            names.add(n.id)
        elif isinstance(n, (ast.Import, ast.ImportFrom)):
            for al in n.names:
                names.add((al.asname or al.name).split(".")[0])
        elif isinstance(n, (ast.Global, ast.Nonlocal)):
            names.update(n.names)
        elif isinstance(n, ast.ExceptHandler) and n.name:
            names.add(n.name)
        stack.extend(ast.iter_child_nodes(n))
    return names


def _undefined(tree):
    module = _bound(ast.Module(body=tree.body, type_ignores=[])) | set(dir(builtins)) | {"__file__", "__name__"}
    bad = []

    def visit(node, scopes):
        for child in ast.iter_child_nodes(node):
            if isinstance(child, (ast.FunctionDef, ast.AsyncFunctionDef, ast.Lambda, ast.ListComp, ast.SetComp,
                                  ast.DictComp, ast.GeneratorExp)):
                visit(child, scopes + [_bound(child)])
            elif isinstance(child, ast.Name) and isinstance(child.ctx, ast.Load):
                if len(scopes) > 1 and not any(child.id in s for s in scopes):
                    bad.append((child.id, child.lineno))
            else:
                visit(child, scopes)

    visit(tree, [module])
    return bad


def test_bench_has_no_undefined_names():
    tree = ast.parse(open(os.path.join(ROOT, "bench.py")).read())
    assert _undefined(tree) == []


def test_checker_catches_an_undefined_name():
    tree = ast.parse("def f(a):\n    x = {'r': small_roof if a else 1}\n    return x\n")
    assert _undefined(tree) == [("small_roof", 2)]


def test_workload_name_is_shared_by_both_arms():
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert src.count('"workload": workload_name(') >= 2      # the libsimplex line and the reference arm
    assert bench.workload_name(8000, 8000, 1) == \
        "dense random LP m=8000 n=8000 FP64 seed 1, slack basis, Dantzig + lowest-index ties"


def test_cpu_baseline_small_and_prefix():
    A, b, c = lpgen.dense_lp(64, 64, 1)
    r = bench.cpu_baseline(A, b, c, 1.0)
    assert r["kind"] == "oracle" and r["cores"] == 1 and r["value"] > 0 and "complete solves" in r["sample"]
    assert r["host"]["nproc"] >= 1
    A, b, c = lpgen.dense_lp(600, 700, 1)
    r = bench.cpu_baseline(A, b, c, 0.5)
    assert r["value"] > 0 and "first" in r["sample"]


def test_golden_prefixes_found():
    pre = bench.golden_prefixes(20000, 40000, 1)
    assert 512 in pre and 4096 in pre
    assert all(os.path.exists(p) for p in pre.values())


def test_host_info_and_pinning():
    before = os.sched_getaffinity(0)
    with bench.pinned_to_one_core() as pin:
        assert os.sched_getaffinity(0) == {pin.core}
        assert pin.host["allowed_cores"] == len(before)
    assert os.sched_getaffinity(0) == before
