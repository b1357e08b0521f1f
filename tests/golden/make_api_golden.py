"""Public API surface of the reference package (names + call signatures),
parsed with ast from /root/reference (no import), for tests/test_api_surface.py.
Modules: the package root and the ones a caller imports by name; cli.py (out
of scope), oracle.py (the reference's own test oracle), and the per-sample
spec / numba internals (kernels.py, factor_sgd.py, core_sgd.py, _loops.py)
are not part of the drop-in surface.

    python tests/golden/make_api_golden.py
"""
import ast
import json
import os

SRC = "/root/reference/pkg/src/sptucker"
MODULES = ["__init__", "coo", "model", "trainer", "estimator", "partition", "counting"]


def sig(fn):
    a = fn.args
    pos = [x.arg for x in a.posonlyargs + a.args]
    kw = [x.arg for x in a.kwonlyargs]
    defaults = {}
    for name, d in zip(pos[len(pos) - len(a.defaults):], a.defaults):
        defaults[name] = ast.unparse(d)
    for x, d in zip(a.kwonlyargs, a.kw_defaults):
        if d is not None:
            defaults[x.arg] = ast.unparse(d)
    return {"args": pos, "kwonly": kw, "defaults": defaults}


out = {}
for mod in MODULES:
    tree = ast.parse(open(os.path.join(SRC, mod + ".py")).read())
    names = {}
    for node in tree.body:
        if isinstance(node, (ast.FunctionDef, ast.ClassDef)) and not node.name.startswith("_"):
            entry = {"kind": "class" if isinstance(node, ast.ClassDef) else "function"}
            if isinstance(node, ast.FunctionDef):
                entry.update(sig(node))
            else:
                methods = {}
                for b in node.body:
                    if isinstance(b, ast.FunctionDef) and (not b.name.startswith("_") or b.name == "__init__"):
                        methods[b.name] = sig(b)
                entry["methods"] = methods
            names[node.name] = entry
        elif isinstance(node, ast.ImportFrom) and mod == "__init__":
            for al in node.names:
                names[al.asname or al.name] = {"kind": "reexport"}
        elif isinstance(node, ast.Assign):
            for tgt in node.targets:
                if isinstance(tgt, ast.Name) and not tgt.id.startswith("_") and tgt.id.isupper():
                    names[tgt.id] = {"kind": "constant"}
    out[mod] = names
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "api_surface.json")
json.dump(out, open(path, "w"), indent=1, sort_keys=True)
print({m: len(v) for m, v in out.items()})
