"""Pins for the oracle's cost model against what the paper fixes (Appendix A).

Sources: tab:flops_breakdown, Appendix A memory footprint and
conv_1d note, §3 footnote, fig:motivation(b) 17.4 GB /
3.3x, SPEC goldens.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import tracegen as tg

M = tg.MODEL_7B
D, N = 4096, 128


def test_spec_layer_goldens():
    t = O.layer_terms(M, 1000)
    assert t["attention_flops"] == 150_601_728_000
    assert t["ssm_flops"] == 209_715_210_000
    assert O.layer_terms(M, 1)["mlp_flops"] == 268_435_456
    assert O.layer_terms(M, 1)["kv_bytes"] == 16_384
    assert t["ssm_state_bytes"] == 1_048_576
    assert t["conv_state_bytes"] == 67_584
    assert O.layer_terms(M, 16)["kv_bytes"] == 262_144      # SPEC:89 (linearity)
    assert O.layer_terms(tg.Model(4, 24, 28, d_state=16), 1)["ssm_state_bytes"] == 131_072  # SPEC:98, N=16 axis
    z = O.layer_terms(M, 0)
    assert z["attention_flops"] == z["ssm_flops"] == z["mlp_flops"] == z["kv_bytes"] == 0


def test_attention_row_flops_per_byte_is_L_plus_2D():
    """tab:flops_breakdown row 3: Attention FLOPs saved per byte = L + 2D,
    = L + 8192 for the 7B.  An attention-only root node's Eq. 1 value
    must equal it exactly (an integer, exact in fp64)."""
    attn1 = tg.Model(1, 0, 0)
    for L in (1, 2, 7, 100, 1000, 4096, 32768, 100_000):
        saved, by, eff = O.node_cost(attn1, 0, L, False)
        assert by == 4 * L * D                      # "4LD" state bytes
        assert eff == L + 2 * D == L + 8192


def test_ssm_row_flops_per_byte():
    """tab:flops_breakdown: SSM FLOPs saved per byte = L (6D/N + 8 + 5/(DN)),
    ~200 L at D=4096, N=128.  With conv excluded (the table omits it,
    PAPER:814) the oracle's double must be the correctly rounded closed form."""
    ssm1 = tg.Model(0, 1, 0, conv_in=0)
    for L in (1, 3, 64, 1000, 32768):
        saved, by, eff = O.node_cost(ssm1, 0, L, True)
        assert by == 2 * D * N                      # "2DN"
        exact = L * (Fraction(6 * D, N) + 8 + Fraction(5, D * N))
        assert eff == float(exact)
        assert abs(eff / L - 200.0) < 1e-5


def test_state_ratio_N_over_2_and_footnote():
    t = O.layer_terms(M, 1)
    # SSM state of one layer vs one token's KVs of one layer: N/2 = 64
    assert Fraction(t["ssm_state_bytes"], t["kv_bytes"]) == N // 2 == 64
    # footnote: d_state / (2 * block_size) = 4 at block 16
    assert Fraction(t["ssm_state_bytes"], O.layer_terms(M, 16)["kv_bytes"]) == 4


def test_conv_share_6_1_percent():
    t = O.layer_terms(M, 1)
    share = t["conv_state_bytes"] / (t["ssm_state_bytes"] + t["conv_state_bytes"])
    assert round(100 * share, 1) == 6.1


def test_fig2b_17_4_GB_and_3_3x():
    """One 10K-token sequence with a state per 16-token block: 17.4 GB and 3.3x
    a same-size Transformer.  Built from the oracle's per-node bytes: 625 stateful nodes."""
    _, node16, _ = O.node_cost(M, 0, 16, True)
    total = 625 * O.node_cost(M, 0, 16, True)[1]
    assert total == 17_397_760_000
    assert round(total / 1e9, 1) == 17.4
    tf = tg.Model(32, 0, 32)  # 7B Transformer: 32 attention layers
    _, kv_tf, _ = O.node_cost(tf, 0, 10_000, False)
    assert round(total / kv_tf, 1) == 3.3


def test_quadratic_identity_and_linearity():
    for L in (1, 5, 1000, 12345):
        a = O.layer_terms(M, L)
        a2 = O.layer_terms(M, 2 * L)
        assert a2["attention_flops"] - 2 * a["attention_flops"] == 8 * L * L * D   # SPEC cost_model invariants
        assert a2["mlp_flops"] == 2 * a["mlp_flops"]
        assert a2["ssm_flops"] == 2 * a["ssm_flops"]


def test_prefill_is_sum_over_layer_types_and_delta_is_parent_relative():
    for L in (0, 1, 100, 1000, 10_000, 32_768):
        t = O.layer_terms(M, L)
        assert O.prefill_flops(M, L) == 4 * t["attention_flops"] + 24 * t["ssm_flops"] + 28 * t["mlp_flops"]
    # a child's savings are relative to its parent's
    s, b, e = O.node_cost(M, 500, 800, True)
    assert s == O.prefill_flops(M, 800) - O.prefill_flops(M, 500)
    assert b == 300 * 65_536 + 26_787_840
    assert e == float(Fraction(s, b))


def test_survey_7b_totals():
    """Values evaluated independently in SURVEY.md §8(c) c.4."""
    assert O.prefill_flops(M, 1) == 13_086_294_256
    assert O.prefill_flops(M, 100) == 1_309_278_232_000
    assert O.prefill_flops(M, 1000) == 13_151_764_720_000
    assert O.prefill_flops(M, 10_000) == 137_415_887_200_000
    assert O.prefill_flops(M, 32_768) == 499_178_286_874_624


def test_fig5_more_ssm_layers_steeper():
    """fig:flops_eff_diff: the more SSM layers, the steeper FLOP efficiency vs L.
    Compare 7B {4,24,28} against a 1:2 hybrid {4,8,12} (single stateful node [0, L))."""
    lo, hi = tg.model_ratio(2), tg.model_ratio(8)
    for L1, L2 in ((1000, 2000), (10_000, 20_000)):
        s_lo = O.node_cost(lo, 0, L2, True)[2] - O.node_cost(lo, 0, L1, True)[2]
        s_hi = O.node_cost(hi, 0, L2, True)[2] - O.node_cost(hi, 0, L1, True)[2]
        assert s_hi > s_lo


def test_zero_byte_node_is_an_error():
    with pytest.raises(O.OracleError):
        O.node_cost(tg.Model(0, 4, 4), 0, 10, False)
