"""pytest plugin: run the REFERENCE's own test modules with this backend
installed (install()) so every by-name prover import in
zklora -- and in the test modules, which import after this plugin has run --
reaches the CUDA path.

    python -m pytest -p dropin_plugin baseline/_ref/zklora_tests/test_sumcheck.py

The reference package itself comes from baseline/_ref (a pip --target install
of /root/reference/pkg; git-ignored, travels to the GPU box with the repo).
At session end the plugin prints how many times each installed backend entry
point was called, so a run that silently bypassed the backend is visible
(tests/test_dropin_reference.py asserts the counts are non-zero)."""

import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (ROOT, REF):
    if p not in sys.path:
        sys.path.insert(0, p)

CALLS = collections.Counter()


def _counted(name, fn):
    def wrapper(*a, **k):
        CALLS[name] += 1
        return fn(*a, **k)

    wrapper.__wrapped__ = fn
    return wrapper


def pytest_configure(config):
    import importlib

    import paper_2508_21393_b200 as zb

    z = importlib.import_module("zklora")
    assert os.path.dirname(z.__file__).startswith(REF), z.__file__
    gpu_commit = os.environ.get("ZKL_DROPIN_GPU_COMMIT") == "1"
    zb.install(z, gpu_commit=gpu_commit)
    # count calls at every installed binding (install() put the backend's
    # functions there; wrap them in place)
    from paper_2508_21393_b200 import gadgets as bg, lookup as bl, nonlinear as bn
    from paper_2508_21393_b200 import sumcheck as bs

    fns = [bs.prove_sumcheck, bl.prove_lookup, bl.compute_multiplicities, bg.prove_matmul,
           bg.prove_elementprod, bn.prove_rescale, bn.prove_swiglu, bn.prove_rsqrt,
           bn.prove_softmax_row]
    if gpu_commit:
        zc = importlib.import_module("zklora.commit")
        fns += [zc.commit, zc.open_batch]  # install()'s dispatchers
    backend = {id(f) for f in fns}
    for m in ("sumcheck", "lookup", "gadgets", "pipeline", "commit"):
        mod = importlib.import_module("zklora." + m)
        for attr, val in list(vars(mod).items()):
            if callable(val) and id(val) in backend:
                setattr(mod, attr, _counted(attr, val))


def pytest_unconfigure(config):
    out = os.environ.get("ZKL_DROPIN_CALLS")
    if out:
        with open(out, "w") as fh:
            json.dump(dict(CALLS), fh)
    sys.stderr.write("dropin backend calls: %s\n" % json.dumps(dict(CALLS), sort_keys=True))
