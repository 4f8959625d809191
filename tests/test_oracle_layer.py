"""CPU pins for oracle/layer.py (NEXT #2: the APB prefill layer around the hot path).

Each step is checked against something other than itself: transformers' LlamaDecoderLayer /
LlamaRMSNorm / LlamaRotaryEmbedding + apply_rotary_pos_emb and torch.nn.functional (library
routines, fp64), closed forms and the rotation invariants of RoPE."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import layer as OL


def _llama(hidden=64, inter=96, hq=4, hk=2, d=16, theta=10000.0, eps=1e-5):
    from transformers import LlamaConfig
    from transformers.models.llama import modeling_llama as ml
    cfg = LlamaConfig(hidden_size=hidden, intermediate_size=inter, num_attention_heads=hq, num_key_value_heads=hk,
                      head_dim=d, rope_theta=theta, rms_norm_eps=eps, attn_implementation="sdpa",
                      max_position_embeddings=8192)
    torch.manual_seed(0)
    layer = ml.LlamaDecoderLayer(cfg, 0).double()
    # transformers' LlamaRMSNorm computes in fp32 even for fp64 inputs; use torch's fused
    # rms_norm (pinned in test_rmsnorm_matches_torch_and_closed_form) so the reference is fp64
    for norm in (layer.input_layernorm, layer.post_attention_layernorm):
        norm.forward = (lambda n: lambda x: torch.nn.functional.rms_norm(x, (x.shape[-1],), n.weight,
                                                                         n.variance_epsilon))(norm)
    with torch.no_grad():
        for p in layer.parameters():
            p.copy_(torch.randn_like(p) * (0.3 if p.ndim == 2 else 0.2) + (1.0 if p.ndim == 1 else 0.0))
    return cfg, layer, ml


def _weights_of(layer, eps, theta):
    a, m = layer.self_attn, layer.mlp
    t = lambda x: x.detach().numpy()
    return {"attn_norm": t(layer.input_layernorm.weight), "ffn_norm": t(layer.post_attention_layernorm.weight),
            "w_qkv": np.concatenate([t(a.q_proj.weight), t(a.k_proj.weight), t(a.v_proj.weight)]),
            "w_o": t(a.o_proj.weight), "w_gu": np.concatenate([t(m.gate_proj.weight), t(m.up_proj.weight)]),
            "w_down": t(m.down_proj.weight), "eps": eps, "theta": theta}


def _cos_sin64(rot, pos, d, theta):
    """fp64 cos/sin in transformers' layout (cat(freqs, freqs)); the library computes them in
    fp32, so only its frequencies are compared (to fp32 rounding) and the angles are redone
    in fp64."""
    inv = theta ** (-np.arange(0, d, 2, dtype=np.float64) / d)
    np.testing.assert_allclose(inv, rot.inv_freq.double().numpy(), rtol=2e-7)
    f = np.asarray(pos, np.float64)[:, None] * inv[None, :]
    emb = torch.from_numpy(np.concatenate([f, f], axis=-1))[None]
    return emb.cos(), emb.sin()


def test_rmsnorm_matches_torch_and_closed_form():
    rng = np.random.default_rng(1)
    x, w = rng.standard_normal((7, 33)), rng.standard_normal(33)
    ref = torch.nn.functional.rms_norm(torch.from_numpy(x), (33,), torch.from_numpy(w), eps=1e-6).numpy()
    np.testing.assert_allclose(OL.rmsnorm(x, w, 1e-6), ref, rtol=1e-13, atol=1e-14)
    # constant row c: c / sqrt(c^2 + eps) * w
    c = 3.0
    np.testing.assert_allclose(OL.rmsnorm(np.full((1, 5), c), np.arange(5.0), 0.5)[0],
                               c / np.sqrt(c * c + 0.5) * np.arange(5.0), rtol=1e-15)


def test_rope_matches_transformers_and_invariants():
    cfg, layer, ml = _llama()
    rng = np.random.default_rng(2)
    rows, heads, d = 9, 3, 16
    x = rng.standard_normal((rows, heads, d))
    pos = np.array([0, 1, 2, 5, 17, 100, 1000, 4095, 3])
    rot = ml.LlamaRotaryEmbedding(cfg)
    xt = torch.from_numpy(x).permute(1, 0, 2)[None]            # [1][heads][rows][d]
    cos, sin = _cos_sin64(rot, pos, d, 10000.0)
    q_ref, _ = ml.apply_rotary_pos_emb(xt, xt, cos, sin)
    np.testing.assert_allclose(OL.rope(x, pos, 10000.0), q_ref[0].permute(1, 0, 2).numpy(), rtol=1e-10, atol=1e-12)
    # position 0 is the identity; every 2-D pair keeps its norm; q.k depends only on p_q - p_k
    np.testing.assert_array_equal(OL.rope(x[:1], [0], 1e4), x[:1])
    y = OL.rope(x, pos, 1e4)
    pair = lambda z: z[..., :8] ** 2 + z[..., 8:] ** 2
    np.testing.assert_allclose(pair(y), pair(x), rtol=1e-12)
    q, k = x[0:1], x[1:2]
    dots = [np.sum(OL.rope(q, [p + 7], 1e4) * OL.rope(k, [p], 1e4)) for p in (0, 3, 250)]
    np.testing.assert_allclose(dots, dots[0], rtol=1e-10)


def test_swiglu_matches_torch():
    rng = np.random.default_rng(3)
    gu = rng.standard_normal((4, 10)) * 4
    g, u = torch.from_numpy(gu[:, :5]), torch.from_numpy(gu[:, 5:])
    np.testing.assert_allclose(OL.swiglu(gu, 5), (torch.nn.functional.silu(g) * u).numpy(), rtol=1e-13)
    assert OL.silu(0.0) == 0.0


@pytest.mark.parametrize("rows", [1, 13])
def test_dense_layer_equals_transformers_llama_layer(rows):
    """H = 1 (plain causal attention): attn_in -> oracle.attention -> attn_out_ffn equals
    transformers' LlamaDecoderLayer in fp64 — pins the RMSNorm, the Q|K|V weight layout, RoPE,
    GQA attention, the O projection, both residuals and the SwiGLU FFN at once."""
    eps, theta = 1e-5, 10000.0
    cfg, layer, ml = _llama(eps=eps, theta=theta)
    lw = _weights_of(layer, eps, theta)
    rng = np.random.default_rng(4)
    x = rng.standard_normal((rows, 64))
    pos = np.arange(rows)
    qkv = OL.attn_in(x, lw, 4, 2, 16, pos, rnd=False)
    O, _ = oracle.attention(qkv[:, :4], qkv[:, 4:6], qkv[:, 6:], 0, np.zeros((0, 2, 16)), np.zeros((0, 2, 16)))
    out = OL.attn_out_ffn(x, O, lw, rnd=False)
    rot = ml.LlamaRotaryEmbedding(cfg)
    xt = torch.from_numpy(x)[None]
    cos, sin = _cos_sin64(rot, pos, 16, theta)
    mask = torch.full((rows, rows), float("-inf"), dtype=torch.float64).triu(1)[None, None]
    with torch.no_grad():
        ref = layer(xt, attention_mask=mask, position_ids=torch.from_numpy(pos)[None],
                    position_embeddings=(cos, sin))
    ref = (ref[0] if isinstance(ref, tuple) else ref)[0].numpy()
    np.testing.assert_allclose(out, ref, rtol=1e-9, atol=1e-10)


def test_apb_layer_single_host_is_dense_layer_and_anchor_rows_are_host_independent():
    """apb_layer with H = 1 equals the dense layer; with H > 1 and l_q = 0 the anchor rows of
    every host (consistent anchor) reproduce host 1's first l_a output rows, since
    anchor queries see only the anchor (G1) at the same starting positions."""
    eps, theta = 1e-5, 10000.0
    cfg, layer, ml = _llama(eps=eps, theta=theta)
    lw = _weights_of(layer, eps, theta)
    rng = np.random.default_rng(5)
    H, l_b, l_a, l_p = 3, 12, 5, 4
    doc = rng.standard_normal((H * l_b, 64))
    retain = {"w1": rng.standard_normal((32, 128)) * 0.1, "b1": None, "w2": rng.standard_normal((4, 32)) * 0.1,
              "b2": None}
    hosts_x = [doc[:l_b]] + [np.concatenate([doc[:l_a], doc[h * l_b:(h + 1) * l_b]]) for h in range(1, H)]
    res = OL.apb_layer(hosts_x, [0] + [l_a] * (H - 1), lw, retain, l_p, 4, 2, 16, rnd=False)
    for h in range(1, H):
        np.testing.assert_allclose(res["out"][h][:l_a], res["out"][0][:l_a], rtol=1e-12, atol=1e-12)
    one = OL.apb_layer([doc[:l_b]], [0], lw, retain, l_p, 4, 2, 16, rnd=False)
    qkv = OL.attn_in(doc[:l_b], lw, 4, 2, 16, np.arange(l_b), rnd=False)
    O, _ = oracle.attention(qkv[:, :4], qkv[:, 4:6], qkv[:, 6:], 0, np.zeros((0, 2, 16)), np.zeros((0, 2, 16)))
    np.testing.assert_allclose(one["out"][0], OL.attn_out_ffn(doc[:l_b], O, lw, rnd=False), rtol=1e-12)


def test_bf16_rounding_points_are_bf16():
    rng = np.random.default_rng(6)
    v = OL.bf16(rng.standard_normal(1000) * 100)
    assert np.array_equal(OL.bf16(v), v)
    bits = synth.f32_to_bf16_bits(v.astype(np.float32))
    assert np.array_equal(synth.bf16_bits_to_f64(bits), v)
