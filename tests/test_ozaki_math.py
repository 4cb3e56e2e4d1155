"""The arithmetic behind the FP64-on-INT8 contraction (csrc/matmul_ozaki.cu), restated with numpy integers: the digit
decomposition is exact, level sums stay inside INT32, truncating the levels gives the stated bound, and the guard of the
auto mode (nothing cut, every non-zero digit pair kept) is exactly the condition for an error-free product.  The GPU kernel
itself is checked against the CPU program in tests/test_gpu_parity.py; this file pins the scheme it implements."""
import numpy as np
import pytest

S = 7


def unit(t):
    """digit t (1-based) has the unit 2^-unit(t): 8-bit digits (csrc/ozaki_digits.cuh)"""
    return 7 + 8 * (t - 1)


def slices(x):
    """rows of x -> (exponents e, signs s, digits d[t] as int64 arrays, remainder r) with x = s 2^e (sum_t d_t 2^-unit(t)) + s 2^e r.
    Every digit is what an int8 holds: the lopsided rounding d = ceil(R - 127/255) keeps what is left inside (c - 1, c] of the
    digit's unit, c = 127/255, so that the next digit is never +128; a row whose largest element is above 127/128 of 2^e is encoded
    negated (s = -1), and when both ends of the row are that large e grows by one."""
    hi, lo = x.max(axis=1), x.min(axis=1)
    mx = np.maximum(np.abs(hi), np.abs(lo))
    e = np.where(mx > 0, np.floor(np.log2(np.maximum(mx, 1e-300))).astype(np.int64) + 1, 0)
    sc = np.exp2(-e.astype(np.float64))
    hi_big, lo_big = hi * sc > 127 / 128, -lo * sc > 127 / 128
    e = e + (hi_big & lo_big)
    sign = np.where(hi_big & ~lo_big, -1.0, 1.0)
    rem = x * (sign * np.exp2(-e.astype(np.float64)))[:, None]
    assert (rem > -1.004).all() and (rem < 0.9961).all()
    digits = []
    for t in range(1, S + 1):
        d = np.rint(rem * 2.0 ** unit(t) + 1.0 / 510.0)
        rem = rem - d * 2.0 ** -unit(t)          # exact in float64
        assert ((d >= -128) & (d <= 127)).all()
        digits.append(d.astype(np.int64))
    return e, sign, digits, rem


def contract(a, bt, c0, keep=S + 1):
    ea, sa, da, _ = slices(a)
    eb, sb, db, _ = slices(bt)
    acc = np.zeros(a.shape[0:1] + bt.shape[0:1])
    for g in range(keep, 1, -1):                     # Horner from the smallest level, as the epilogue does
        level = sum(da[t - 1] @ db[g - t - 1].T for t in range(1, S + 1) if 1 <= g - t <= S)
        assert np.abs(level).max() < 2 ** 31         # INT32 accumulators
        acc = acc / 256.0 + level
    return c0 + sa[:, None] * sb[None, :] * np.ldexp(acc, (ea[:, None] + eb[None, :] - 14).astype(np.int64))


def app_operands(n):
    i = np.arange(n, dtype=np.float64)
    return (i[:, None] + i[None, :]) / n, (i[None, :] - i[:, None]) / n      # a, bt = b^T


@pytest.mark.parametrize("n", [128, 256])
def test_application_operands_use_two_digits_and_the_product_is_exact(n):
    a, bt = app_operands(n)
    for x in (a, bt):
        _, _, d, rem = slices(x)
        assert (rem == 0).all() and all((dt == 0).all() for dt in d[2:])     # log2(N) + 2 bits: digits 1 and 2 only, so even the
        # 6-slice form (digits <= 6, pairs t + u <= 7) keeps every non-zero pair: the cheapest error-free form of auto mode
    i = np.arange(n, dtype=np.float64)
    s1, s2 = n * (n - 1) / 2, (n - 1) * n * (2 * n - 1) / 6
    closed = (s2 + (i[:, None] - i[None, :]) * s1 - n * i[:, None] * i[None, :]) / n ** 2
    assert np.array_equal(contract(a, bt, np.zeros((n, n))), closed)


def test_random_operands_meet_the_stated_bound():
    rs = np.random.RandomState(0)
    n = 192
    a = rs.uniform(-1, 1, (n, n)) * np.exp2(rs.randint(-30, 30, (n, 1)))
    bt = rs.uniform(-1, 1, (n, n)) * np.exp2(rs.randint(-30, 30, (n, 1)))
    c0 = rs.uniform(-1, 1, (n, n))
    got = contract(a, bt, c0)
    exact = (c0.astype(np.longdouble) + a.astype(np.longdouble) @ bt.astype(np.longdouble).T)
    err = np.abs(got.astype(np.longdouble) - exact).astype(np.float64)
    stated = (S + 3) * n * 2.0 ** (-7 * S) * np.abs(a).max(axis=1)[:, None] * np.abs(bt).max(axis=1)[None, :]
    ulp = 2.0 ** -52 * np.abs(exact).astype(np.float64)                      # the final rounding of c itself
    assert (err <= stated + ulp).all()
    bar = 1e-12 * (np.abs(c0) + np.abs(a) @ np.abs(bt).T)
    assert (err <= 0.05 * bar).all()                                         # far inside the norm-wise tolerance


def test_guard_condition_is_the_error_free_condition():
    rs = np.random.RandomState(1)
    n = 96
    c0 = np.zeros((n, n))

    def top(x):
        _, _, d, rem = slices(x)
        return (rem != 0).any(), max((t + 1 for t in range(S) if (d[t] != 0).any()), default=0)

    # 21-bit integers: nothing cut, 3 + 3 digits -> every pair kept -> exact
    a, bt = (rs.randint(-2 ** 20, 2 ** 20, (n, n)).astype(np.float64) for _ in range(2))
    (cut_a, ta), (cut_b, tb) = top(a), top(bt)
    assert not cut_a and not cut_b and ta + tb <= S + 1
    assert np.array_equal(contract(a, bt, c0), a @ bt.T)
    # 33-bit integers: nothing cut, but 5 + 5 digits: pairs beyond level 8 are dropped -> not exact, the guard says so
    a, bt = (rs.randint(-2 ** 32, 2 ** 32, (n, n)).astype(np.float64) for _ in range(2))
    (cut_a, ta), (cut_b, tb) = top(a), top(bt)
    assert not cut_a and not cut_b and ta + tb > S + 1
    exact = a.astype(np.int64).astype(object) @ bt.astype(np.int64).astype(object).T
    assert (contract(a, bt, c0).astype(object) != exact).any()
    # full-mantissa doubles of mixed magnitude (seven digits reach 54 bits below the row maximum): elements are cut
    assert top(rs.uniform(-1, 1, (n, n)) * np.exp2(-rs.randint(0, 20, (n, n)).astype(np.float64)))[0]


# ---- the forms of the persistent kernel (matmul_ozaki.cu: <SA, SB, LV>) and the rule that picks one -------------------------

FORMS = [(2, 2, 3), (3, 2, 4), (2, 3, 4), (3, 3, 5), (4, 3, 6), (3, 4, 6), (4, 4, 7), (5, 5, 5), (6, 6, 6), (7, 7, 7)]


def pairs_of(form):
    sa, sb, lv = form
    return {(t, u) for t in range(1, sa + 1) for u in range(1, sb + 1) if t + u <= lv + 1}


def test_rectangular_form_reproduces_the_product_exactly():
    """Digits a_1..a_SA against b_1..b_SB, every pair: when no operand has a digit beyond (SA, SB) the level sums, weighted
    2^-(unit(t) + unit(u)), are the exact product -- with integers only."""
    rs = np.random.RandomState(5)
    k = 96
    for sa, sb in ((2, 2), (3, 2), (2, 3), (4, 4)):
        a = rs.randint(-(2 ** (7 * sa - 1)) + 1, 2 ** (7 * sa - 1), (8, k)).astype(np.float64)
        b = rs.randint(-(2 ** (7 * sb - 1)) + 1, 2 ** (7 * sb - 1), (8, k)).astype(np.float64)
        ea, sa_, da, ra = slices(a)
        eb, sb_, db, rb = slices(b)
        assert not ra.any() and not rb.any()
        assert not any(d.any() for d in da[sa:]) and not any(d.any() for d in db[sb:])   # nothing beyond the form's digits
        total = np.zeros((8, 8), dtype=object)
        for t in range(1, sa + 1):
            for u in range(1, sb + 1):
                level = da[t - 1].astype(np.int64) @ db[u - 1].astype(np.int64).T
                assert np.abs(level).max() < 2 ** 31
                total = total + level.astype(object) * 2 ** (2 * unit(S) - unit(t) - unit(u))      # common denominator 2^(2 unit(S))
        exact = a.astype(np.int64).astype(object) @ b.astype(np.int64).astype(object).T
        scale = np.array([[int(p) * int(q) * 2 ** (int(x) + int(y)) for y, q in zip(eb, sb_)] for x, p in zip(ea, sa_)], dtype=object)
        assert (total * scale == exact * 2 ** (2 * unit(S))).all()


def test_pick_form_takes_the_cheapest_error_free_form():
    from paper_1806_01430_b200 import capi
    for ta in range(0, 9):
        for tb in range(0, 9):
            got = capi.gene8_pick_form(False, ta, tb)
            need = {(t, u) for t in range(1, max(ta, 1) + 1) for u in range(1, max(tb, 1) + 1)}
            ok = [f for f in FORMS if need <= pairs_of(f)]
            if not ok:
                assert got == 0, (ta, tb, got)
                continue
            form = (got // 100, got // 10 % 10, got % 10)
            assert form in ok, (ta, tb, got)
            assert len(pairs_of(form)) == min(len(pairs_of(f)) for f in ok), (ta, tb, got)
            assert capi.gene8_pick_form(True, ta, tb) == 0                # anything cut: the FP64 pipe
