"""The reference's OWN hot-path test modules, run unmodified against this
backend through install().

baseline/_ref holds a pip --target install of /root/reference/pkg (plus its
tests under baseline/_ref/zklora_tests); it is git-ignored and travels to the
GPU box with the repo snapshot.  Each module runs in a fresh interpreter with
tests/dropin_plugin.py, which installs the backend before the module imports
its provers and reports how many times each backend entry point ran.

The hypothesis seed is fixed: test_pipeline.py::test_random_configs_prove_and_verify
can draw configurations on which the reference's OWN witness generation
raises RangeViolation (gadgets.py:575; the pure reference reproduces it with
layers=1, seq=2, dim=4, mlp=4, vocab=4, rank=1, seed=3198), which has nothing
to do with the prover under test."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "zklora_tests")

# module -> backend entry points that must have run
MODULES = {
    "test_field.py": [],
    "test_mle.py": [],
    "test_sumcheck.py": ["prove_sumcheck"],
    "test_lookup.py": ["prove_lookup", "compute_multiplicities"],
    "test_gadgets.py": ["prove_matmul", "prove_elementprod", "prove_rescale", "prove_swiglu",
                        "prove_rsqrt", "prove_softmax_row"],
    "test_pipeline.py": ["prove_matmul", "prove_elementprod", "prove_rescale"],
}


# with install(gpu_commit=True): the reference's commit / open_batch calls go to
# the GPU Hyrax implementation (commit_gpu.py) as well
GPU_COMMIT_MODULES = {
    "test_commit.py": ["commit", "open_batch"],
    "test_lookup.py": ["prove_lookup", "commit", "open_batch"],
    "test_gadgets.py": ["prove_matmul", "commit", "open_batch"],
    "test_pipeline.py": ["prove_matmul", "commit", "open_batch"],
}


def _run_module(module, tmp_path, gpu_commit):
    calls = tmp_path / "calls.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join(
        [os.path.join(ROOT, "tests"), os.path.join(ROOT, "baseline", "_ref"), ROOT]),
        ZKL_DROPIN_CALLS=str(calls), ZKL_DROPIN_GPU_COMMIT="1" if gpu_commit else "0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "dropin_plugin",
                        "-p", "no:cacheprovider", "--hypothesis-seed=0", "--rootdir", REF_TESTS,
                        os.path.join(REF_TESTS, module)],
                       cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=3000)
    return r, calls


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="baseline/_ref not installed")
@pytest.mark.parametrize("module", sorted(GPU_COMMIT_MODULES))
def test_reference_module_passes_with_gpu_commitments(module, tmp_path):
    r, calls = _run_module(module, tmp_path, True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    counts = json.loads(calls.read_text())
    for name in GPU_COMMIT_MODULES[module]:
        assert counts.get(name, 0) > 0, (name, counts)


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="baseline/_ref not installed")
@pytest.mark.parametrize("module", sorted(MODULES))
def test_reference_module_passes_on_backend(module, tmp_path):
    calls = tmp_path / "calls.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join(
        [os.path.join(ROOT, "tests"), os.path.join(ROOT, "baseline", "_ref"), ROOT]),
        ZKL_DROPIN_CALLS=str(calls))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "dropin_plugin",
                        "-p", "no:cacheprovider", "--hypothesis-seed=0", "--rootdir", REF_TESTS,
                        os.path.join(REF_TESTS, module)],
                       cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=3000)
    tail = (r.stdout[-3000:] + r.stderr[-2000:])
    assert r.returncode == 0, tail
    counts = json.loads(calls.read_text())
    for name in MODULES[module]:
        assert counts.get(name, 0) > 0, (name, counts)
