"""CPU model of the int8 seed's digit arithmetic (csrc/seed_i8.cu), test
infrastructure only: the encodings are exact, the 21 kept digit-pair products
reproduce an fp64 product to ~1e-13 relative (Frobenius), and the int32
accumulator bounds the kernel relies on hold.  numpy integer arithmetic is exact,
so this pins the scheme independently of the GPU."""
import numpy as np

MAGIC = 2.0 ** 52 + sum(128 * 256 ** k for k in range(6))


def balanced_digits(x, e):
    """fma(x, 2^(46-e), 2^52 + sum 128 256^k): bytes of the low 48 mantissa bits,
    xor 0x80 -> signed digits d_k (k = 0 least significant)."""
    u = x * 2.0 ** (46 - e) + MAGIC  # exact in fp64 for |x| <= 2^e (one rounding, as the DFMA)
    bits = u.view(np.uint64) & np.uint64((1 << 48) - 1)
    d = [((bits >> np.uint64(8 * k)) & np.uint64(0xFF)).astype(np.int64) - 128 for k in range(6)]
    return d


def value(d):
    return sum(dk * 256 ** k for k, dk in enumerate(d))


def test_digits_reconstruct_the_rounded_value():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(100000)
    e = int(np.frexp(np.abs(x).max())[1])
    d = balanced_digits(x, e)
    for dk in d:
        assert dk.min() >= -128 and dk.max() <= 127
    assert np.abs(d[5]).max() <= 65  # top digit of |v| <= 2^46
    v = np.rint(x * 2.0 ** (46 - e)).astype(np.int64)
    assert np.array_equal(value(d), v)


def seed_model(Y, KR, kept=5):
    """Right seed Y @ KR through digits: per-column KR scale, one Y scale, diagonals
    a + b <= kept (top-first), exact int64 sums, Horner in fp64."""
    ey = int(np.frexp(np.abs(Y).max())[1])
    yd = balanced_digits(Y.ravel(), ey)
    yd = [d.reshape(Y.shape) for d in yd][::-1]  # top first
    out = np.zeros((Y.shape[0], KR.shape[1]))
    for r in range(KR.shape[1]):
        er = int(np.frexp(np.abs(KR[:, r]).max())[1])
        kd = balanced_digits(KR[:, r].copy(), er)[::-1]
        diag = [np.zeros(Y.shape[0], dtype=np.int64) for _ in range(6)]
        for a in range(6):
            for b in range(6 - a):
                if a + b <= kept:
                    diag[a + b] += yd[a] @ kd[b]
        assert max(np.abs(dd).max() for dd in diag) < 2 ** 31
        h = diag[0].astype(np.float64)
        for dd in diag[1:]:
            h = h * 256.0 + dd
        out[:, r] = h * 2.0 ** (ey + er - 52)
    return out


def test_21_pairs_reach_1e12():
    rng = np.random.default_rng(2)
    Y = rng.standard_normal((96, 128))
    KR = rng.standard_normal((128, 6)) * rng.standard_normal((128, 6))
    want = Y @ KR
    got = seed_model(Y, KR)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 1e-12, err
    # dropping one more diagonal (15 pairs) loses the fp64 gate
    err15 = np.linalg.norm(seed_model(Y, KR, kept=4) - want) / np.linalg.norm(want)
    assert err15 > 1e-12


def test_integer_inputs_are_exact():
    Y = np.arange(1, 9, dtype=float).reshape(2, 4)
    KR = np.ones((4, 2))
    assert np.array_equal(seed_model(Y, KR), Y @ KR)
