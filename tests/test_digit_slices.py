"""The digit-slice arithmetic of the int8 tensor-core Gram (csrc/gram_i8.cu), restated
in numpy: exact balanced 7-bit digits, and the truncated slice-product sum reproducing
x_j x_k to the FP64 rounding level.  Documents the kernel's numerics without a GPU."""
import numpy as np


def digits(x, e, S=8):
    """As i8_slice_kernel: N = rint(x 2^(6+7(S-1)-e)) (|N| <= 2^55), then N's balanced base-128
    digits from the bottom, d = ((N + 64) mod 128) - 64, N <- (N - d) / 128; the top digit
    is what remains.  x 2^(6-e) = sum_s d_s 2^(-7(s-1)) + rest, |rest| <= 2^(-7(S-1)-1)."""
    sh = 7 * S - 1
    N = np.rint(np.ldexp(x, sh - e)).astype(np.int64)
    out = [None] * S
    for s in range(S - 1, 0, -1):
        d = ((N + 64) & 127) - 64
        N = (N - d) >> 7
        out[s] = d
    out[0] = N
    rest = np.ldexp(x, sh - e) - np.rint(np.ldexp(x, sh - e))
    return np.array(out).astype(np.float64), rest


def slice_dot(xj, xk, S):
    """The kernel's sum over s + t <= S + 1 of d_s d_t 2^(-7(s+t-2)) (exact int32 groups,
    smallest weight first), scaled back by 2^(e_j + e_k - 12)."""
    _, ej = np.frexp(np.abs(xj).max())
    _, ek = np.frexp(np.abs(xk).max())
    dj, _ = digits(xj, ej, S)
    dk, _ = digits(xk, ek, S)
    total = 0.0
    for w in range(S + 1, 1, -1):
        cw = sum(int(np.dot(dj[s - 1].astype(np.int64), dk[w - s - 1].astype(np.int64))) for s in range(1, w))
        assert abs(cw) < 2 ** 31
        total += np.ldexp(float(cw), -7 * (w - 2))
    return np.ldexp(total, ej + ek - 12)


def test_digits_are_exact_and_balanced():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(10000) * 10.0 ** rng.uniform(-20, 20, 10000)
    _, e = np.frexp(np.abs(x).max())
    d, rest = digits(x, e)
    assert np.all(np.abs(d) <= 64)
    assert np.all(np.abs(rest) <= 0.5)            # rounding x 2^(55-e) to an integer
    # exact reconstruction in integer arithmetic (Python ints): the digits plus the rest
    scale = [2 ** (7 * (8 - s)) for s in range(1, 9)]     # digit s weight, in units of 2^-49
    for i in range(0, 10000, 997):
        acc = sum(int(d[s, i]) * scale[s] for s in range(8))
        v = np.ldexp(x[i], 6 - e + 49)                       # exact power-of-two scaling
        assert abs(v - acc) <= 0.5 + 1e-12               # the rest is below half a unit of 2^-49


def test_truncated_slice_products_match_the_product():
    """sum over s + t <= 9 of d_s d_t 2^(-7(s+t-2)), scaled back, vs x_j x_k."""
    rng = np.random.default_rng(1)
    xj, xk = rng.standard_normal(5000), rng.standard_normal(5000)
    _, ej = np.frexp(np.abs(xj).max())
    _, ek = np.frexp(np.abs(xk).max())
    dj, _ = digits(xj, ej)
    dk, _ = digits(xk, ek)
    total = 0.0
    for w in range(9, 1, -1):                            # smallest weight first, as the kernel
        cw = sum(int(np.dot(dj[s - 1].astype(np.int64), dk[w - s - 1].astype(np.int64))) for s in range(1, w))
        assert abs(cw) < 2 ** 31                          # one int32 accumulator per group
        total += np.ldexp(float(cw), -7 * (w - 2))
    g = np.ldexp(total, ej + ek - 12)
    exact = float(np.dot(xj.astype(np.longdouble), xk.astype(np.longdouble)))
    bound = 2.0 ** -52 * np.linalg.norm(xj) * np.linalg.norm(xk)
    assert abs(g - exact) <= bound


def test_seven_slices_stay_at_the_fp64_tile_level():
    """S = 7 (chosen by i8_colexp_kernel while every column's max/rms <= 8): 28 slice products.
    Each entry stays within the worst-case bound 2^-45.8 max|x_j| max|x_k| per sample, and on
    Gaussian columns the error relative to |x_j||x_k| is at the FP64 DMMA tiles' level
    (2e-15 .. 2e-14 measured); S = 8 matches an FP64 dot product."""
    rng = np.random.default_rng(3)
    m = 5000
    X = rng.standard_normal((m, 12))
    err = {7: [], 8: []}
    for j in range(12):
        for k in range(j, 12):
            exact = float(np.dot(X[:, j].astype(np.longdouble), X[:, k].astype(np.longdouble)))
            nrm = np.linalg.norm(X[:, j]) * np.linalg.norm(X[:, k])
            for S in (7, 8):
                e = abs(slice_dot(X[:, j], X[:, k], S) - exact)
                worst = 2.0 ** (-45.8 if S == 7 else -52.8) * m * np.abs(X[:, j]).max() * np.abs(X[:, k]).max()
                assert e <= worst
                err[S].append(e / nrm)
    assert max(err[7]) <= 1e-14
    assert max(err[8]) <= 1e-15
