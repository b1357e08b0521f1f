"""Drop-in check: every public name of the reference package's caller-facing
modules (tests/golden/api_surface.json, parsed from the reference by
tests/golden/make_api_golden.py) exists here under the same module name, with
the same positional / keyword parameter names (extensions may only append
parameters that have defaults) and the same literal defaults."""

import importlib
import inspect
import json
import os

import pytest

HERE = os.path.join(os.path.dirname(__file__), "golden")
SURFACE = json.load(open(os.path.join(HERE, "api_surface.json")))
CASES = [(mod, name) for mod, names in sorted(SURFACE.items()) for name in sorted(names)]


def _ours(mod):
    return importlib.import_module("paper_2204_07104_b200" + ("" if mod == "__init__" else "." + mod))


def _check_sig(fn, want, label):
    if isinstance(fn, property):
        return
    params = inspect.signature(fn).parameters
    pos = [p.name for p in params.values() if p.kind in (p.POSITIONAL_ONLY, p.POSITIONAL_OR_KEYWORD)]
    kw = [p.name for p in params.values() if p.kind == p.KEYWORD_ONLY]
    n = len(want["args"])
    assert pos[:n] == want["args"], f"{label}: positional parameters {pos} != {want['args']}"
    for extra in pos[n:]:
        assert params[extra].default is not inspect.Parameter.empty, f"{label}: added parameter {extra} needs a default"
    assert kw[:len(want["kwonly"])] == want["kwonly"], f"{label}: keyword-only parameters {kw} != {want['kwonly']}"
    for name, src in want["defaults"].items():
        try:
            ref = eval(src, {"__builtins__": {}}, {})  # literals and simple expressions only
        except Exception:
            continue
        got = params[name].default
        assert got is not inspect.Parameter.empty, f"{label}: {name} has no default"
        assert got == ref, f"{label}: default {name}={got!r} != {ref!r}"


@pytest.mark.parametrize("mod,name", CASES)
def test_reference_name_exists_with_same_signature(mod, name):
    want = SURFACE[mod][name]
    ours = _ours(mod)
    assert hasattr(ours, name), f"{mod}.{name} missing"
    obj = getattr(ours, name)
    if want["kind"] == "function":
        _check_sig(obj, want, f"{mod}.{name}")
    elif want["kind"] == "class":
        for meth, sig in want.get("methods", {}).items():
            assert hasattr(obj, meth), f"{mod}.{name}.{meth} missing"
            _check_sig(inspect.getattr_static(obj, meth), sig, f"{mod}.{name}.{meth}")
