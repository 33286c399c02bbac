"""The LoRA-block proof schedule (paper_2508_21393_b200/block.py) on the GPU,
checked byte for byte against the reference's own gadget provers run through
the same schedule (tests/golden/block.json, written by make_golden.py
gen_block with RefBlockProver)."""

import pytest

from conftest import FIELDS, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2508_21393_b200 import block as BK  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402
from paper_2508_21393_b200.transcript import Transcript  # noqa: E402


def _tiny(g):
    seq, hidden, heads, hd, ffn, rank, lora = g["shape"]
    shape = BK.BlockShape("tiny", seq, hidden, heads, hd, ffn, rank, tuple(lora))
    gm, z, a, en, eps = g["fp"]
    return shape, BK.FixedPoint(gamma_fp=gm, zeta=z, act_bound=a, exp_n=en, eps=eps)


@pytest.mark.parametrize("field", ["big", "test"])
def test_tiny_block_matches_reference_gadgets(field):
    g = load_golden("block.json")
    shape, fp = _tiny(g)
    c = [c for c in g["cases"] if c["field"] == field][0]
    p = FIELDS[field]
    tables = BK.block_tables(D.spec_for(p), fp)
    w = BK.BlockWitness(shape, seed=c["seed"], fp=fp, device="cuda")
    tr = Transcript(b"zkl/golden/block", p, field.encode())
    assert tr.state.hex() == c["state_before"]
    P = BK.prove_block(w, BK.BlockProver(tr, tables))
    assert P.log == c["log"]
    assert P.clipped == c["clipped"]
    assert tr.state.hex() == c["state_end"]
    s = BK.summary(P)
    assert s["total"]["count"] == len(c["log"])


@pytest.mark.parametrize("field", ["big"])
def test_tiny_block_witness_pass_then_replay_matches(field):
    """WitnessRecorder + replay proves exactly what the interleaved schedule
    proves (same gadget log, same end transcript state as the reference)."""
    g = load_golden("block.json")
    shape, fp = _tiny(g)
    c = [c for c in g["cases"] if c["field"] == field][0]
    p = FIELDS[field]
    tables = BK.block_tables(D.spec_for(p), fp)
    w = BK.BlockWitness(shape, seed=c["seed"], fp=fp, device="cuda")
    rec = BK.prove_block(w, BK.WitnessRecorder(tables))
    tr = Transcript(b"zkl/golden/block", p, field.encode())
    P = rec.replay(BK.BlockProver(tr, tables))
    assert P.log == c["log"] and P.clipped == c["clipped"]
    assert tr.state.hex() == c["state_end"]
