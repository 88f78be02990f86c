"""Host restatement of the grid epoch's fixed-point exchange arithmetic
(paper_1911_07722_b200/csrc/epoch_grid.cu: fexp60, inv_scale, the
(value << 8) + 1 accumulator words and their decode).  No GPU: these are the
integer identities the kernel relies on -- order independence, the
completion count in the low byte, exact differences modulo 2^64, and the
Cauchy-Schwarz scales keeping every sum inside 55 bits."""
import numpy as np
import pytest

MASK64 = (1 << 64) - 1


def fexp60(v):
    """Biased fp32 exponent of a non-negative value, floored at 2^-60."""
    e = int(np.float32(v).view(np.int32)) >> 23
    return max(e, 67)


def inv_scale(ea, eb):
    """2^-shift for a value bounded by sqrt(A B), A < 2^(ea-126), B < 2^(eb-126)."""
    field = 127 - 52 + ((ea + eb - 251) >> 1)
    assert 1 <= field <= 254, "scale must be a normal fp32 power of two"
    return np.int32(field << 23).view(np.float32)


def encode(partial, scale):
    f = np.float32(partial) * np.float32(scale)
    assert abs(float(f)) < 2.0 ** 54
    fx = int(np.rint(np.float64(f)))
    return ((fx << 8) + 1) & MASK64


def decode(cur, prev, g):
    diff = (cur - prev) & MASK64
    assert diff & 0xFF == g & 0xFF
    if diff >= 1 << 63:
        diff -= 1 << 64
    return diff >> 8  # arithmetic shift: the count byte drops out


@pytest.mark.parametrize("seed", range(5))
def test_accumulator_is_order_independent_and_never_reset(seed):
    g = np.random.default_rng(seed)
    G = 145
    word = int(g.integers(0, 1 << 63)) * 2 + 1  # arbitrary state left by earlier events
    for _ in range(40):  # 40 events through the same slot
        partials = (g.standard_normal(G) * 10.0 ** g.uniform(-3, 3)).astype(np.float32)
        scale = np.float32(2.0 ** 30)
        words = [encode(p, scale) for p in partials]
        want = sum(int(np.rint(np.float64(np.float32(p) * scale))) for p in partials)
        prev = word
        totals = set()
        for _perm in range(3):
            w = prev
            seen_complete_early = False
            for k, i in enumerate(g.permutation(G)):
                if k > 0 and ((w - prev) & 0xFF) == (G & 0xFF):
                    seen_complete_early = True
                w = (w + words[i]) & MASK64
            assert not seen_complete_early  # the count only matches after all G adds
            totals.add(decode(w, prev, G))
        assert totals == {want}
        word = w


@pytest.mark.parametrize("seed", range(4))
def test_scales_keep_sums_inside_55_bits(seed):
    g = np.random.default_rng(100 + seed)
    rows, G = 4096, 16
    for _ in range(50):
        cs = 10.0 ** g.uniform(-12, 12)
        ws = 10.0 ** g.uniform(-12, 12)
        x = (g.standard_normal(rows) * cs).astype(np.float32)
        xk = (g.standard_normal(rows) * 10.0 ** g.uniform(-12, 12)).astype(np.float32)
        w = (g.standard_normal(rows) * ws).astype(np.float32)
        q_e = np.float32(np.dot(x.astype(np.float64), x.astype(np.float64)))
        q_k = np.float32(np.dot(xk.astype(np.float64), xk.astype(np.float64)))
        qmax = max(q_e, q_k)
        # the kernel's bound on ||w||^2: d * max|w|^2 (>= the true norm)
        w2 = np.float32(rows) * np.float32(np.abs(w).max()) ** 2
        if not (np.isfinite(q_e) and np.isfinite(q_k) and np.isfinite(w2)):
            continue
        sc_s = 1.0 / float(inv_scale(fexp60(q_e), fexp60(w2)))
        sc_g = 1.0 / float(inv_scale(fexp60(q_e), fexp60(qmax)))
        parts_s = [float(np.dot(x[i::G].astype(np.float64), w[i::G].astype(np.float64)))
                   for i in range(G)]
        parts_g = [float(np.dot(x[i::G].astype(np.float64), xk[i::G].astype(np.float64)))
                   for i in range(G)]
        for parts, sc in ((parts_s, sc_s), (parts_g, sc_g)):
            assert all(abs(p) * sc < 2.0 ** 52 for p in parts)
            assert sum(abs(p) for p in parts) * sc < 2.0 ** 52  # Cauchy-Schwarz over the slices
            total = sum(int(np.rint(p * sc)) for p in parts)
            assert abs(total) < 1 << 54
            # resolution: the fixed-point total is within G/2 units of the exact sum
            assert abs(total / sc - sum(parts)) <= (G / 2 + 1) / sc


def test_zero_and_tiny_bounds_stay_normal():
    for a in (0.0, 1e-45, 2.0 ** -60, 1.0, 3e38, np.inf):
        for b in (0.0, 2.0 ** -60, 1.0, 3e38):
            s = inv_scale(fexp60(a), fexp60(b))
            assert np.isfinite(s) and s > 0
            assert float(np.float32(0.0) * (np.float32(1.0) / s)) == 0.0
