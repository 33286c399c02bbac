"""The LoRA-block proof schedule (paper_2508_21393_b200/block.py) on the GPU:

* byte for byte against the reference's own gadget provers run through the
  same schedule (tests/golden/block.json, make_golden.py gen_block);
* judged by the reference's own verifiers in the loop (harness/refverify.py:
  every gadget, with independent checks of every opened value), which must
  accept the honest block and reject a tampered witness;
* at full LLaMA-2-7B / 13B shape: the witness pass raises RangeViolation
  rather than clip, so a completed pass means every quotient is in range."""

import os
import sys

import pytest

from conftest import FIELDS, ROOT, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2508_21393_b200 import block as BK  # noqa: E402
from paper_2508_21393_b200 import device as D  # noqa: E402
from paper_2508_21393_b200.transcript import Transcript  # noqa: E402

sys.path.insert(0, ROOT)
from harness import refverify as RV  # noqa: E402

needs_ref = pytest.mark.skipif(not RV.reference_available(), reason="baseline/_ref not installed")


def _tiny(g):
    seq, hidden, heads, hd, ffn, rank, lora = g["shape"]
    shape = BK.BlockShape("tiny", seq, hidden, heads, hd, ffn, rank, tuple(lora))
    return shape, BK.FixedPoint(**g["fp"])


def _witness(g, c, device="cuda"):
    shape, fp = _tiny(g)
    return BK.BlockWitness(shape, seed=c["seed"], fp=fp, device=device, wstd=g["wstd"],
                           dy_std=g["dy_std"]), fp


@pytest.mark.parametrize("field", ["big", "test"])
def test_tiny_block_matches_reference_gadgets(field):
    g = load_golden("block.json")
    c = [c for c in g["cases"] if c["field"] == field][0]
    p = FIELDS[field]
    w, fp = _witness(g, c)
    tables = BK.block_tables(D.spec_for(p), fp)
    tr = Transcript(b"zkl/golden/block", p, field.encode())
    assert tr.state.hex() == c["state_before"]
    P = BK.prove_block(w, BK.BlockProver(tr, tables))
    assert P.log == c["log"]
    assert tr.state.hex() == c["state_end"]
    s = BK.summary(P)
    assert s["total"]["count"] == len(c["log"])


@pytest.mark.parametrize("field", ["big"])
def test_tiny_block_witness_pass_then_replay_matches(field):
    """WitnessRecorder + replay proves exactly what the interleaved schedule
    proves (same gadget log, same end transcript state as the reference)."""
    g = load_golden("block.json")
    c = [c for c in g["cases"] if c["field"] == field][0]
    p = FIELDS[field]
    w, fp = _witness(g, c)
    tables = BK.block_tables(D.spec_for(p), fp)
    rec = BK.prove_block(w, BK.WitnessRecorder(tables))
    tr = Transcript(b"zkl/golden/block", p, field.encode())
    P = rec.replay(BK.BlockProver(tr, tables))
    assert P.log == c["log"]
    assert tr.state.hex() == c["state_end"]


@needs_ref
@pytest.mark.parametrize("field", ["big", "test"])
def test_tiny_block_reference_verifiers_accept(field):
    g = load_golden("block.json")
    c = [c for c in g["cases"] if c["field"] == field][0]
    p = FIELDS[field]
    w, fp = _witness(g, c)
    spec = D.spec_for(p)
    tables = BK.block_tables(spec, fp)
    P, s = RV.prove_and_verify_block(w, tables, spec, b"zkl/golden/block", field.encode())
    assert s["transcripts_equal"], s
    assert s["rejected"] == 0 and s["opening_mismatches"] == 0, s
    assert s["gadgets_verified"] == len(c["log"]) and s["openings_unchecked"] == 0, s
    assert s["verifier_accept"]


@needs_ref
def test_tiny_block_tampered_quotient_rejected(monkeypatch):
    """One narrowed entry off by one (the kind of witness a clamped quotient
    gives): the reference verify_rescale rejects at that gadget."""
    g = load_golden("block.json")
    c = [c for c in g["cases"] if c["field"] == "big"][0]
    p = FIELDS["big"]
    w, fp = _witness(g, c)
    spec = D.spec_for(p)
    tables = BK.block_tables(spec, fp)
    real = BK._divmod
    calls = {"n": 0}

    def tampered(wide, divisor, fp_):
        q, r = real(wide, divisor, fp_)
        calls["n"] += 1
        if calls["n"] == 5:
            q = q.clone()
            q.view(-1)[0] += 1
        return q, r

    monkeypatch.setattr(BK, "_divmod", tampered)
    P, s = RV.prove_and_verify_block(w, tables, spec, b"zkl/golden/block", b"big")
    assert not s["verifier_accept"]
    assert s["first_rejected"][0] == "rescale", s


@needs_ref
def test_tiny_block_tampered_lookup_output_rejected(monkeypatch):
    """A wrong SiLU output (not the table's value) is an unprovable lookup:
    the multiplicity histogram raises ElementNotInTable before any proof."""
    from paper_2508_21393_b200.lookup import ElementNotInTable

    g = load_golden("block.json")
    c = [c for c in g["cases"] if c["field"] == "big"][0]
    w, fp = _witness(g, c)
    tables = BK.block_tables(D.spec_for(FIELDS["big"]), fp)
    real = BK._lut

    def bad(table_y, x, x0):
        out = real(table_y, x, x0).clone()
        out.view(-1)[3] += 1
        return out

    monkeypatch.setattr(BK, "_lut", bad)
    tr = Transcript(b"zkl/golden/block", FIELDS["big"], b"big")
    with pytest.raises(ElementNotInTable):
        BK.prove_block(w, BK.BlockProver(tr, tables))


@pytest.mark.parametrize("shape", ["7b", "13b"])
def test_llama_block_witness_in_range(shape):
    """Full-size witness pass (bench seed): completes, so no quotient leaves
    quant_range and no residual add leaves int16 (they raise)."""
    sh = {"7b": BK.LLAMA2_7B, "13b": BK.LLAMA2_13B}[shape]
    tables = BK.block_tables(D.spec_for(FIELDS["big"]))
    w = BK.BlockWitness(sh, seed=1)
    rec = BK.prove_block(w, BK.WitnessRecorder(tables))
    kinds = [c[0] for c in rec.calls]
    assert kinds.count("rescale_w") > 40 and kinds.count("matadd") > 10
    del rec, w
    torch.cuda.empty_cache()
