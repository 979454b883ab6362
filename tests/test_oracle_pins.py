"""Pins for the fp64 oracle against things other than itself (CPU only).

Each test names the passage / invariant it pins.
A plausible mistake in the oracle (dropped scale, wrong GQA map, exclusive
causal boundary, log base, merge weights, sign) fails at least one of these.
"""
import math
import random

import numpy as np
import pytest
import torch

from oracle import attention, attention_group, merge, partial, NEG_INF
import synth


def _rand(shape, rng, amp=1.0):
    # bf16-representable values (as the GPU would see them)
    x = torch.from_numpy(rng.standard_normal(shape).astype(np.float32) * amp)
    return x.to(torch.bfloat16).double().numpy()


def _brute(q, k, v, q_pos, key_pos, scale):
    """Independent pure-Python brute force: full score matrix, -inf mask,
    math.fsum row sums (S:138 'naive double-loop implementation')."""
    T, h_q, d = q.shape
    N, h_kv, _ = k.shape
    G = h_q // h_kv
    o = np.zeros((T, h_q, d))
    lse = np.full((T, h_q), -np.inf)
    for t in range(T):
        for h in range(h_q):
            g = h // G
            z = []
            for j in range(N):
                if key_pos[j] <= q_pos[t]:
                    z.append(scale * math.fsum(float(q[t, h, e]) * float(k[j, g, e]) for e in range(d)))
                else:
                    z.append(-math.inf)
            m = max(z)
            if m == -math.inf:
                continue
            p = [math.exp(zz - m) if zz != -math.inf else 0.0 for zz in z]
            l = math.fsum(p)
            for e in range(d):
                o[t, h, e] = math.fsum(p[j] * float(v[j, g, e]) for j in range(N)) / l
            lse[t, h] = m + math.log(l)
    return o, lse


@pytest.mark.parametrize("case", range(12))
def test_oracle_vs_bruteforce_fsum(case):
    """random tiny cases match a naive double-loop to 1e-12 relative."""
    rng = np.random.default_rng(100 + case)
    h_kv = int(rng.choice([1, 2]))
    G = int(rng.choice([1, 2, 4]))
    h_q = h_kv * G
    d = int(rng.choice([8, 16]))
    N = int(rng.integers(1, 40))
    T = int(rng.integers(1, 6))
    q = _rand((T, h_q, d), rng, 2.0)
    k = _rand((N, h_kv, d), rng)
    v = _rand((N, h_kv, d), rng)
    q_pos = np.sort(rng.integers(-2, N + 2, size=T))      # includes fully-masked rows
    key_pos = np.arange(N)
    scale = 1.0 / math.sqrt(d)
    o, lse = attention(q, k, v, q_pos, key_pos, scale)
    ob, lb = _brute(q, k, v, q_pos, key_pos, scale)
    np.testing.assert_allclose(o, ob, rtol=1e-12, atol=1e-14)
    fin = np.isfinite(lb)
    assert np.array_equal(fin, np.isfinite(lse))
    np.testing.assert_allclose(lse[fin], lb[fin], rtol=1e-12, atol=1e-14)
    assert np.all(o[~fin] == 0.0)


@pytest.mark.parametrize("G", [1, 4, 8])
def test_oracle_vs_torch_sdpa_bottom_right(G):
    """Textbook library routine: torch fp64 SDPA with an explicit bottom-right
    causal mask (is_causal is top-left when L != S) and enable_gqa (h // G map)."""
    rng = np.random.default_rng(7 + G)
    h_kv, d, N, c = 2, 32, 50, 13
    h_q = h_kv * G
    q = _rand((c, h_q, d), rng, 3.0)
    k = _rand((N, h_kv, d), rng)
    v = _rand((N, h_kv, d), rng)
    q_pos = np.arange(N - c, N)           # chunk = last c tokens (prefix N-c)
    o, lse = attention(q, k, v, q_pos)
    qt = torch.from_numpy(q).permute(1, 0, 2)[None]
    kt = torch.from_numpy(k).permute(1, 0, 2)[None]
    vt = torch.from_numpy(v).permute(1, 0, 2)[None]
    mask = torch.ones(c, N, dtype=torch.bool).tril(N - c)
    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=mask, enable_gqa=True)
    np.testing.assert_allclose(o, ref[0].permute(1, 0, 2).numpy(), rtol=1e-10, atol=1e-12)
    # logsumexp of the masked scaled scores
    kk = torch.from_numpy(k).repeat_interleave(G, dim=1)
    s = torch.einsum("thd,jhd->thj", torch.from_numpy(q), kk) / math.sqrt(d)
    s = s.masked_fill(~mask[:, None, :], -math.inf)
    np.testing.assert_allclose(lse, torch.logsumexp(s, dim=-1).numpy(), rtol=1e-12)


def test_gqa_map_is_contiguous_not_interleaved():
    """Reading R2: kv_head = h // G.  The interleaved map h % h_kv must differ."""
    rng = np.random.default_rng(3)
    h_kv, G, d, N = 2, 4, 16, 20
    q = _rand((1, h_kv * G, d), rng, 2.0)
    k = _rand((N, h_kv, d), rng)
    v = _rand((N, h_kv, d), rng)
    o, _ = attention(q, k, v, [N - 1])
    for h in range(h_kv * G):
        og, _ = attention_group(q[:, h:h + 1], k[:, h // G], v[:, h // G], [N - 1], np.arange(N), 1 / math.sqrt(d))
        np.testing.assert_allclose(o[:, h], og[:, 0], rtol=1e-13, atol=1e-15)
    o_bad = np.stack([attention_group(q[:, h:h + 1], k[:, h % h_kv], v[:, h % h_kv], [N - 1], np.arange(N),
                                      1 / math.sqrt(d))[0][:, 0] for h in range(h_kv * G)], axis=1)
    assert np.abs(o_bad - o).max() > 1e-3


def test_gqa_equals_repeated_kv_mha():
    """I3 (north_star): GQA equals MHA with each KV head repeated G times."""
    rng = np.random.default_rng(11)
    h_kv, G, d, N, T = 2, 4, 16, 33, 5
    q = _rand((T, h_kv * G, d), rng, 2.0)
    k = _rand((N, h_kv, d), rng)
    v = _rand((N, h_kv, d), rng)
    qp = np.arange(N - T, N)
    o, lse = attention(q, k, v, qp)
    o2, lse2 = attention(q, np.repeat(k, G, axis=1), np.repeat(v, G, axis=1), qp)
    np.testing.assert_allclose(o, o2, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(lse, lse2, rtol=1e-13)


def test_single_key_identity():
    """I4: one visible key => O = V_j, LSE = z_j."""
    rng = np.random.default_rng(5)
    d = 16
    q = _rand((1, 1, d), rng)
    k = _rand((1, 1, d), rng)
    v = _rand((1, 1, d), rng)
    o, lse = attention(q, k, v, [0])
    np.testing.assert_array_equal(o[0, 0], v[0, 0])
    assert lse[0, 0] == pytest.approx(float(q[0, 0] @ k[0, 0]) / math.sqrt(d), rel=1e-15)


def test_identical_keys_give_prefix_mean():
    """I5: identical K rows => O = mean of the visible V rows."""
    rng = np.random.default_rng(6)
    N, d = 30, 16
    q = _rand((3, 2, d), rng, 4.0)
    k = np.repeat(_rand((1, 1, d), rng), N, axis=0)
    v = _rand((N, 1, d), rng)
    qp = [4, 17, 29]
    o, _ = attention(q, k, v, qp)
    for i, p in enumerate(qp):
        for h in range(2):
            np.testing.assert_allclose(o[i, h], v[:p + 1, 0].mean(axis=0), rtol=1e-13, atol=1e-15)


def test_closed_form_k_zero():
    """I12: K = 0 => O[t] = mean(V[0..pos]), LSE = ln(pos+1)."""
    rng = np.random.default_rng(8)
    N, d = 257, 8
    q = _rand((4, 4, d), rng, 8.0)
    k = np.zeros((N, 1, d))
    v = _rand((N, 1, d), rng)
    qp = [0, 63, 128, 256]
    o, lse = attention(q, k, v, qp)
    for i, p in enumerate(qp):
        np.testing.assert_allclose(o[i], np.broadcast_to(v[:p + 1, 0].mean(0), (4, d)), rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(lse[i], math.log(p + 1), rtol=1e-14)


def test_closed_form_needle_across_shards():
    """I13: K_j* = alpha q, others 0 => O = (e^{z*} V_j* + sum_{j!=j*} V_j) / (e^{z*} + n - 1);
    needle in a non-tail shard so the merge decides."""
    rng = np.random.default_rng(9)
    N, d, js = 200, 16, 37
    q = _rand((1, 1, d), rng)
    k = np.zeros((N, 1, d))
    k[js, 0] = 0.5 * q[0, 0]
    v = _rand((N, 1, d), rng)
    s = 1 / math.sqrt(d)
    zs = s * float(k[js, 0] @ q[0, 0])
    want = (math.exp(zs) * v[js, 0] + (v[:, 0].sum(0) - v[js, 0])) / (math.exp(zs) + N - 1)
    o, lse = attention(q, k, v, [N - 1])
    np.testing.assert_allclose(o[0, 0], want, rtol=1e-12)
    assert lse[0, 0] == pytest.approx(math.log(math.exp(zs) + N - 1), rel=1e-13)
    parts = [partial(q, k, v, [N - 1], (a, b)) for a, b in [(0, 64), (64, 128), (128, 200)]]
    om, lm = merge(parts)
    np.testing.assert_allclose(om[0, 0], want, rtol=1e-12)


def test_convex_hull_and_affine_equivariance():
    """I6 outputs are convex combinations; I7 O(aV+b) = aO(V)+b."""
    rng = np.random.default_rng(10)
    N, d = 64, 8
    q = _rand((6, 2, d), rng, 4.0)
    k = _rand((N, 1, d), rng)
    v = _rand((N, 1, d), rng)
    qp = np.array([3, 10, 20, 40, 50, 63])
    o, _ = attention(q, k, v, qp)
    for i, p in enumerate(qp):
        lo = v[:p + 1, 0].min(0)
        hi = v[:p + 1, 0].max(0)
        assert np.all(o[i] >= lo[None] - 1e-12) and np.all(o[i] <= hi[None] + 1e-12)
    o2, _ = attention(q, k, 3.0 * v - 1.25, qp)
    np.testing.assert_allclose(o2, 3.0 * o - 1.25, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(25))
def test_merge_any_partition_equals_unsharded(seed):
    """I1 (north_star; S:155 random splits p in {2,4,8}, n <= 256, within 1e-6),
    including empty parts and permutations (1e-9)."""
    rng = random.Random(seed)
    nrng = np.random.default_rng(seed)
    h_kv = rng.choice([1, 2])
    G = rng.choice([1, 2, 4, 8])
    d = rng.choice([8, 16, 32])
    N = rng.randint(1, 256)
    T = rng.randint(1, 8)
    q = _rand((T, h_kv * G, d), nrng, 2.0)
    k = _rand((N, h_kv, d), nrng)
    v = _rand((N, h_kv, d), nrng)
    qp = np.sort(nrng.integers(0, N, size=T))
    o, lse = attention(q, k, v, qp)
    P = rng.choice([1, 2, 4, 8])
    cuts = sorted(rng.randint(0, N) for _ in range(P - 1))
    bounds = list(zip([0] + cuts, cuts + [N]))         # may contain empty shards
    parts = [partial(q, k, v, qp, b) for b in bounds]
    om, lm = merge(parts)
    np.testing.assert_allclose(om, o, rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(lm, lse, rtol=1e-12)
    perm = list(range(P))
    rng.shuffle(perm)
    op, lp = merge([parts[i] for i in perm])
    np.testing.assert_allclose(op, om, rtol=1e-9, atol=1e-14)
    np.testing.assert_allclose(lp, lm, rtol=1e-12)


def test_merge_identity_and_empty_part_noop():
    """S:154 merge of one part is the identity; I8 an (0, -inf) part is a no-op;
    R7 all-empty rows merge to (0, -inf) without NaN."""
    rng = np.random.default_rng(12)
    o = rng.standard_normal((5, 3, 8))
    l = rng.standard_normal((5, 3))
    om, lm = merge([(o, l)])
    np.testing.assert_allclose(om, o, rtol=1e-15)
    np.testing.assert_allclose(lm, l, rtol=1e-15)
    e = (np.zeros_like(o), np.full_like(l, NEG_INF))
    om2, lm2 = merge([e, (o, l), e])
    np.testing.assert_allclose(om2, o, rtol=1e-15)
    np.testing.assert_allclose(lm2, l, rtol=1e-15)
    oz, lz = merge([e, e])
    assert np.all(oz == 0) and np.all(np.isneginf(lz))
    with pytest.raises(ValueError):
        merge([])
    with pytest.raises(ValueError):
        merge([(o, l), (o[:, :2], l[:, :2])])


def test_merge_weights_are_natural_log():
    """Reading R5: LSE at the boundary is a natural log.  Two parts with
    lse 0 and ln 3 weigh 1/4 and 3/4."""
    o1 = np.zeros((1, 2))
    o2 = np.ones((1, 2))
    om, lm = merge([(o1, np.array([0.0])), (o2, np.array([math.log(3.0)]))])
    np.testing.assert_allclose(om, [[0.75, 0.75]], rtol=1e-15)
    assert lm[0] == pytest.approx(math.log(4.0), rel=1e-15)


def test_partial_state_equals_spec_representation():
    """R6 / S:123-128: (o, lse) equals SPEC's (unnormalised o, max, denominator)
    via lse = m + ln l and o = o_unnorm / l, computed by brute force."""
    rng = np.random.default_rng(13)
    N, d = 40, 8
    q = _rand((1, 1, d), rng, 4.0)
    k = _rand((N, 1, d), rng)
    v = _rand((N, 1, d), rng)
    o, lse = partial(q, k, v, [N - 1], (10, 30))
    z = [float(q[0, 0] @ k[j, 0]) / math.sqrt(d) for j in range(10, 30)]
    m = max(z)
    w = [math.exp(x - m) for x in z]
    den = math.fsum(w)
    un = np.array([math.fsum(w[i] * v[10 + i, 0, e] for i in range(20)) for e in range(d)])
    assert lse[0, 0] == pytest.approx(m + math.log(den), rel=1e-14)
    np.testing.assert_allclose(o[0, 0], un / den, rtol=1e-13)


def test_chunked_prefill_equals_one_shot():
    """I2 (north_star): chunked prefill with any chunk size (each chunk sees only
    the prefix + itself) equals one-shot causal prefill."""
    rng = np.random.default_rng(14)
    n, h_kv, G, d = 97, 1, 4, 16
    q = _rand((n, h_kv * G, d), rng, 2.0)
    k = _rand((n, h_kv, d), rng)
    v = _rand((n, h_kv, d), rng)
    o_full, l_full = attention(q, k, v, np.arange(n))
    for c in (1, 7, 32, 64, 97):
        outs, lses = [], []
        for a in range(0, n, c):
            b = min(n, a + c)
            oc, lc = attention(q[a:b], k[:b], v[:b], np.arange(a, b))
            outs.append(oc)
            lses.append(lc)
        np.testing.assert_allclose(np.concatenate(outs), o_full, rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(np.concatenate(lses), l_full, rtol=1e-13)


def test_decode_is_last_prefill_row_and_mask_leak():
    """I9 decode = last row of prefill; I10 changing K/V beyond q_pos leaves
    O bit-identical."""
    rng = np.random.default_rng(15)
    n, d = 50, 16
    q = _rand((n, 4, d), rng, 2.0)
    k = _rand((n, 1, d), rng)
    v = _rand((n, 1, d), rng)
    o_full, l_full = attention(q, k, v, np.arange(n))
    od, ld = attention(q[-1:], k, v, [n - 1])
    np.testing.assert_array_equal(od[0], o_full[-1])
    qp = [20]
    o1, l1 = attention(q[20:21], k, v, qp)
    k2, v2 = k.copy(), v.copy()
    k2[21:] = 1e3
    v2[21:] = np.nan
    o2, l2 = attention(q[20:21], k2, v2, qp)
    np.testing.assert_array_equal(o1, o2)
    np.testing.assert_array_equal(l1, l2)


def test_lse_is_log_of_total_visible_mass():
    """I11: LSE(merged) = ln sum over all visible e^z (fsum brute force)."""
    rng = np.random.default_rng(16)
    N, d = 120, 8
    q = _rand((1, 1, d), rng, 4.0)
    k = _rand((N, 1, d), rng)
    v = _rand((N, 1, d), rng)
    parts = [partial(q, k, v, [99], b) for b in [(0, 30), (30, 90), (90, 120)]]
    _, lm = merge(parts)
    tot = math.fsum(math.exp(float(q[0, 0] @ k[j, 0]) / math.sqrt(d)) for j in range(100))
    assert lm[0, 0] == pytest.approx(math.log(tot), rel=1e-13)


def test_dimension_errors():
    with pytest.raises(ValueError):
        attention(np.zeros((1, 4, 8)), np.zeros((3, 1, 16)), np.zeros((3, 1, 16)), [2])
    with pytest.raises(ValueError):
        attention(np.zeros((1, 3, 8)), np.zeros((3, 2, 8)), np.zeros((3, 2, 8)), [2])


def test_oracle_on_synth_block_streaming_matches_small_blocks():
    """Blocking of the oracle's dot products does not change the result beyond
    fp64 regrouping of the value sum."""
    K = synth.kv_block(1, synth.STREAM_K, 0, 3000, 1, 64).double().numpy()[:, 0]
    V = synth.kv_block(1, synth.STREAM_V, 0, 3000, 1, 64).double().numpy()[:, 0]
    q = synth.queries(1, 1, 4, 64).double().numpy()
    a = attention_group(q, K, V, [2999], np.arange(3000), 0.125, block=65536)
    b = attention_group(q, K, V, [2999], np.arange(3000), 0.125, block=97)
    np.testing.assert_allclose(a[0], b[0], rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(a[1], b[1], rtol=1e-15)
