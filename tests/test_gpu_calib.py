"""the stage-2 calibration step on the GPU (mobi_joint_step, csrc/calib.cu) against the
oracle's restatement of trainer::joint_forward / joint_backward (trainer.hpp:203-263, 341-396), itself
pinned to the compiled reference in tests/test_oracle.py.  fp64 throughout; the GPU's GEMMs sum in a
different order (and use FMA) than the reference's loops, so parity is to 1e-9 of each output's scale
(measured differences are ~1e-14), except the per-group clip sums, which keep the reference's order."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from test_oracle import JOINT_KEYS, assert_joint_close, joint_case

pytestmark = pytest.mark.gpu


def run_gpu(c, sched, t, force=False, backward=True):
    from paper_2602_20191_b200 import joint_step
    d = {k: (torch.from_numpy(np.ascontiguousarray(v)).cuda() if k in ("w", "w1", "b1", "w2", "b2", "x", "y_fp") else v)
         for k, v in c.items()}
    r = joint_step(**d, sched=sched, t=t, force_gates_on=force, backward=backward)
    return {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in r.items()}


@pytest.mark.parametrize("sched,t,force", [((8.0, 3.0, 10, 0, 1e-3), 4, False),   # soft gates, log schedule
                                          ((8.0, 3.0, 10, 0, 1e-3), 10, False),  # t = L: indicator gates
                                          ((6.0, 2.5, 7, 2, 1e-2), 3, False),    # cosine
                                          ((6.0, 2.5, 7, 3, 1e-2), 5, False),    # exponential
                                          ((8.0, 3.0, 10, 1, 1e-3), 2, True)])   # force_gates_on ablation
def test_joint_step_matches_oracle(sched, t, force):
    c = joint_case()
    assert_joint_close(run_gpu(c, sched, t, force), O.joint_step_np(**c, sched=sched, t=t, force_gates_on=force))


@pytest.mark.parametrize("bits", [(4, 2, 2), (2, 3, 3), (1, 1, 1, 1, 1, 1, 1, 1)])
def test_joint_step_slice_layouts(bits):
    c = joint_case(slice_bits=bits, seed=11)
    sched = (8.0, 3.0, 12, 1, 1e-3)
    assert_joint_close(run_gpu(c, sched, 5), O.joint_step_np(**c, sched=sched, t=5))


def test_joint_step_larger_layer_and_forward_only():
    """Several 64x64 GEMM tiles in every dimension, ragged edges (out 200, in 330, T 150, h 70)."""
    c = joint_case(out=200, inn=330, T=150, h=70, gs=128, seed=2)
    sched = (8.0, 3.0, 20, 0, 1e-4)
    assert_joint_close(run_gpu(c, sched, 7), O.joint_step_np(**c, sched=sched, t=7))
    f = run_gpu(c, sched, 7, backward=False)
    assert "d_w1" not in f
    assert_joint_close(f, O.joint_step_np(**c, sched=sched, t=7, backward=False))


def test_joint_step_deterministic():
    c = joint_case(out=130, inn=256, T=90, h=40, seed=4)
    sched = (8.0, 3.0, 10, 0, 1e-3)
    a, b = run_gpu(c, sched, 3), run_gpu(c, sched, 3)
    for k in JOINT_KEYS:
        assert np.array_equal(a[k], b[k]), k
    assert a["loss"] == b["loss"]


def test_joint_step_errors_like_reference():
    from paper_2602_20191_b200 import MobiInvalidArgument
    c = joint_case()
    with pytest.raises(MobiInvalidArgument, match=r"outside \[1,10\]"):
        run_gpu(c, (8.0, 3.0, 10, 0, 1e-3), 0)
    with pytest.raises(O.OracleError, match=r"outside \[1,10\]"):
        O.reference().joint_step(**c, sched=(8.0, 3.0, 10, 0, 1e-3), t=0)


@pytest.mark.parametrize("bits", [(2, 2, 2, 2), (4, 2, 2), (3, 5)])
def test_msb_step_matches_oracle(bits):
    """Stage 1 (trainer.hpp:404-426): mobi_msb_step against the oracle."""
    from paper_2602_20191_b200 import msb_step
    c = joint_case(out=150, inn=330, T=70, slice_bits=bits, seed=13)
    cuda = {k: torch.from_numpy(c[k]).cuda() for k in ("w", "x", "y_fp")}
    r = msb_step(cuda["w"], c["group_size"], bits[0], c["gamma_lo"], c["gamma_hi"], cuda["x"], cuda["y_fp"])
    ref = O.msb_step_np(w=c["w"], group_size=c["group_size"], slice_bits=bits, gamma_lo=c["gamma_lo"],
                        gamma_hi=c["gamma_hi"], x=c["x"], y_fp=c["y_fp"])
    assert abs(r["loss"] - ref["loss"]) <= 1e-9 * ref["loss"]
    y = r["y_msb"].cpu().numpy()
    assert np.abs(y - ref["y_msb"]).max() <= 1e-9 * np.abs(ref["y_msb"]).max()
    for k in ("d_gamma_lo", "d_gamma_hi"):
        assert np.abs(r[k] - ref[k]).max() <= 1e-9 * np.abs(ref[k]).max(), k


@pytest.mark.parametrize("out,inn,T,h,gs,bits", [(5, 7, 1, 1, 128, (4, 4)),      # gs > in, one token, h = 1
                                                 (9, 130, 3, 2, 64, (2, 2, 2, 2)),  # partial group, tiny tiles
                                                 (129, 65, 17, 65, 32, (3, 3, 2))])  # tile edges + 1
def test_joint_and_msb_step_edge_shapes(out, inn, T, h, gs, bits):
    c = joint_case(out=out, inn=inn, T=T, h=h, gs=gs, slice_bits=bits, seed=21)
    sched = (8.0, 3.0, 10, 0, 1e-3)
    assert_joint_close(run_gpu(c, sched, 4), O.joint_step_np(**c, sched=sched, t=4))
    from paper_2602_20191_b200 import msb_step
    r = msb_step(torch.from_numpy(c["w"]).cuda(), gs, bits[0], c["gamma_lo"], c["gamma_hi"],
                 torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y_fp"]).cuda())
    ref = O.msb_step_np(w=c["w"], group_size=gs, slice_bits=bits, gamma_lo=c["gamma_lo"], gamma_hi=c["gamma_hi"],
                        x=c["x"], y_fp=c["y_fp"])
    assert abs(r["loss"] - ref["loss"]) <= 1e-9 * ref["loss"]
    for k in ("d_gamma_lo", "d_gamma_hi"):
        assert np.abs(r[k] - ref[k]).max() <= 1e-9 * max(np.abs(ref[k]).max(), 1e-300), k
