"""The two joiner-backward modes (D20).

The CTA-pair joiner forward stores every row's P~ with one offset m_ref (the max of the row's first
32 logits of V tiles 0 and 1); pruned_combine then folds the blank / label picks into P~ and the
joiner backward runs as plain GEMMs (K10: dh = sc_r (P~' W), K11: d_w = P~'^T (sc_r h_r)).  A logit more
than 60 above m_ref anywhere in a row sends the whole batch to the per-(row, tile) rescaling path.
Both must match the oracle; rnnt_pruned_backward_mode reports which one ran.
"""
import numpy as np
import pytest
import torch

import synth
from synth import f32_to_bf16_bits
import paper_2206_13236_b200 as R
from gpu_common import assert_bf16_grad, assert_loss, dims_of_batch, oracle_h_bits, to_dev

pytestmark = pytest.mark.gpu


def _run(b, h_bits, ranges):
    dev = to_dev(b)
    d = dims_of_batch(b)
    o = R.alloc_outputs(d, "cuda")
    ws = torch.empty(R.rnnt_workspace_bytes(d), dtype=torch.uint8, device="cuda")
    h = torch.from_numpy(np.ascontiguousarray(h_bits).view(np.int16)).cuda()
    rg = torch.from_numpy(np.ascontiguousarray(ranges, np.int32)).cuda()
    R.rnnt_pruned_loss(h, dev["w_out"], dev["b_out"], dev["symbols"], rg, dev["boundary"], d, 1.0,
                       o["loss_pruned"], o["d_enc"], o["d_dec"], o["d_w"], o["d_b"], o["status"], ws)
    plain = R.rnnt_pruned_backward_mode(d, ws)
    torch.cuda.synchronize()
    return plain, {k: o[k].cpu().numpy() for k in ("loss_pruned", "d_enc", "d_dec", "d_w", "d_b")}


def _check(b, want_plain):
    from test_gpu_parity import _oracle_pruned, check_ranges, check_simple
    g, o = check_simple(b)
    ranges = check_ranges(b, o)
    plain, got = _run(b, oracle_h_bits(b, ranges), ranges)
    assert plain == want_plain, f"backward mode: plain={plain}, expected {want_plain}"
    ref = _oracle_pruned(b, ranges)
    assert_loss(got["loss_pruned"], ref["loss"], "loss_pruned")
    for k in ("d_w", "d_b", "d_enc", "d_dec"):
        assert_bf16_grad(got[k], ref[k], k)


def _spiked(v_spike, value=80.0, V=400, J=32):
    b = synth.make_custom([60, 41, 17], [20, 12, 16], V, J, 5, seed=41, logit_scale=2.0)
    if v_spike is not None:
        b.b_out_bits = b.b_out_bits.copy()
        b.b_out_bits[v_spike] = f32_to_bf16_bits(np.array([value], np.float32))[0]
    return b


def test_plain_mode_default():
    """Ordinary logits: one offset per row, plain GEMM backward."""
    _check(_spiked(None), True)


@pytest.mark.parametrize("v_spike", [5, 140])
def test_spike_inside_reference_columns_stays_plain(v_spike):
    """A bias spike inside the reference columns (the first 32 of V tiles 0 / 1) raises m_ref itself."""
    _check(_spiked(v_spike), True)


@pytest.mark.parametrize("v_spike", [40, 300, 399])
def test_spike_beyond_reference_falls_back(v_spike):
    """A logit ~80 above m_ref in a later chunk / tile: that tile takes its own offset and the
    backward rescales P~ per (row, tile)."""
    _check(_spiked(v_spike), False)


def test_c2_shard_plain():
    """A 4-utterance shard of config 2 (V = 500, J = 512): the bench workload's shapes."""
    from test_gpu_guards import _sub
    _check(_sub(synth.make_batch(2), [0, 1, 2, 3]), True)


@pytest.mark.parametrize("J", [64, 32])
def test_large_v_plain(J):
    """V >= 6144: the precomputed Hs and (J % 64 == 0) the CTA-pair d_w kernel; J = 32: the wide kernel."""
    _check(_spiked(None, V=6500, J=J), True)


@pytest.mark.parametrize("J", [64, 32])
def test_large_v_rescale(J):
    """V >= 6144 with a spike beyond the reference columns: the wide kernel's rescaling mode (the pair
    kernel, launched alongside, must leave it alone)."""
    _check(_spiked(5000, V=6500, J=J), False)


def test_prepare_split_matches():
    """rnnt_pruned_loss_prepare + rnnt_pruned_loss_forward_prepared (the prepare call on its own stream, as
    step(RNNT_SPLIT_PREP=1) runs it) give bit-identical results to rnnt_pruned_loss_forward."""
    from test_gpu_guards import _sub
    from test_gpu_parity import check_ranges, check_simple
    b = _sub(synth.make_batch(2), [0, 1, 2, 3])
    g, o = check_simple(b)
    ranges = check_ranges(b, o)
    h_bits = oracle_h_bits(b, ranges)
    dev = to_dev(b)
    d = dims_of_batch(b)
    h = torch.from_numpy(np.ascontiguousarray(h_bits).view(np.int16)).cuda()
    rg = torch.from_numpy(np.ascontiguousarray(ranges, np.int32)).cuda()
    res = []
    for split in (False, True):
        out = R.alloc_outputs(d, "cuda")
        ws = torch.full((R.rnnt_workspace_bytes(d),), 0xFF, dtype=torch.uint8, device="cuda")
        if split:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            R.rnnt_pruned_loss_prepare(rg, dev["symbols"], dev["boundary"], d, dev["b_out"], 1.0, ws, side)
            torch.cuda.current_stream().wait_stream(side)
            R.rnnt_pruned_loss_forward_prepared(h, dev["w_out"], dev["b_out"], dev["symbols"], rg, dev["boundary"], d,
                                                1.0, out["loss_pruned"], out["status"], ws)
        else:
            R.rnnt_pruned_loss_forward(h, dev["w_out"], dev["b_out"], dev["symbols"], rg, dev["boundary"], d, 1.0,
                                       out["loss_pruned"], out["status"], ws)
        R.rnnt_pruned_loss_backward_input(h, dev["w_out"], rg, dev["boundary"], d, out["d_enc"], out["d_dec"], ws)
        R.rnnt_pruned_loss_backward_weight(h, d, out["d_w"], out["d_b"], ws)
        torch.cuda.synchronize()
        res.append({k: out[k].cpu().numpy() for k in ("loss_pruned", "d_enc", "d_dec", "d_w", "d_b")})
    for k in res[0]:
        assert np.array_equal(res[0][k], res[1][k]), k
