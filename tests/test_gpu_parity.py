"""GPU parity: libmhg.so (tcgen05 kind::i8 path) vs the CPU oracle / reference.

Integer work mod q: the bar is bit-exact equality of the WHOLE output
container (Matrix::operator==, matrix.hpp:30-33) wherever the oracle can
finish in seconds; at benchmark sizes, size-independent checks (Freivalds'
identity over the whole result + dense recompute of sampled output tiles that
cover every top-level Morton quadrant and the view's edges and corners).
"""
import numpy as np
import pytest

from oracle.binding import OP_ADD, OP_SET, OP_SUB, Views

pytestmark = pytest.mark.gpu


def reference_available():
    import os

    from oracle.binding import REF_SO
    return os.path.exists(REF_SO)

P16 = 65521
P31 = 2147483647
P24 = 16777213  # a 24-bit prime: three limbs


def _containers(mh, n, t, q, cells):
    lay, mod = mh.Layout(n, t), mh.Modulus(q)
    return [mh.Matrix(lay, mod).upload(c) for c in cells]


def _run_gpu(mh, n, t, q, out, lhs, rhs, v: Views, op):
    A, B, Cm = _containers(mh, n, t, q, (out, lhs, rhs))
    prob = mh.Problem(mh.Sub(A, v.out_origin, v.rows, v.cols),
                      mh.Sub(B, v.lhs_origin, v.rows, v.inner),
                      mh.Sub(Cm, v.rhs_origin, v.inner, v.cols))
    ctr = mh.mm(prob, op)
    got = A.cells()
    return got, ctr


def _random_views(rng, n, r=None, k=None, c=None):
    r = r or int(rng.integers(1, n + 1))
    k = k or int(rng.integers(1, n + 1))
    c = c or int(rng.integers(1, n + 1))
    return r, k, c, [int(rng.integers(0, n - d + 1)) for d in (r, c, r, k, k, c)]


def _views_from(oracle, n, t, r, k, c, corners):
    ia, ja, ib, jb, ic, jc = corners
    return Views(oracle.encode(n, t, ia, ja), oracle.encode(n, t, ib, jb),
                 oracle.encode(n, t, ic, jc), r, k, c)


def _fill(oracle, seed, n, q):
    g = oracle.rng(seed)
    return [oracle.fill_below(g, n * n, q) for _ in range(3)]


def test_smoke_cfg1_shape(gpu, mh, oracle, reference):
    """BASELINE cfg1: n=512, t=32, p=65521, C = A*B, full aligned views."""
    n, t, q = 512, 32, P16
    out, lhs, rhs = _fill(oracle, 0, n, q)
    out[:] = 0
    v = Views(0, 0, 0, n, n, n)
    got, ctr = _run_gpu(mh, n, t, q, out, lhs, rhs, v, OP_ADD)
    want = out.copy()
    ref_ctr = reference.mm_oblivious(n, t, q, want, lhs, rhs, v)
    assert np.array_equal(got, want)
    assert ctr.as_tuple() == ref_ctr.as_tuple()


# limb-count boundaries (251 / 257: 1 -> 2 limbs; 65519 / 65537: 2 -> 3; 16777213 /
# 16777259: 3 -> 4) and a 2-limb prime whose 2^16 mod q >= 256 (40961: the per-class fold
# instead of the lean one, no early TMEM release)
@pytest.mark.parametrize("q", [2, 97, 251, 257, 40961, 65519, P16, 65537, P24, 16777259, 1000003, P31])
@pytest.mark.parametrize("op", [OP_ADD, OP_SUB, OP_SET])
def test_random_misaligned_views(gpu, mh, oracle, q, op):
    """Random (ragged, misaligned, rectangular) views; whole-container equality."""
    rng = np.random.default_rng(q * 7 + op)
    for it in range(6):
        n = int(rng.choice([64, 128, 256]))
        t = int(rng.choice([x for x in (4, 8, 16, 32, 64) if x <= n]))
        r, k, c, corners = _random_views(rng, n)
        v = _views_from(oracle, n, t, r, k, c, corners)
        out, lhs, rhs = _fill(oracle, 1000 + it, n, q)
        got, _ = _run_gpu(mh, n, t, q, out, lhs, rhs, v, op)
        want = out.copy()
        oracle.mm_dense(n, t, q, want, lhs, rhs, v, op=op)
        assert np.array_equal(got, want), (n, t, q, op, v)


@pytest.mark.parametrize("n,t", [(48, 3), (96, 6), (192, 12), (64, 2), (320, 10), (384, 24)])
def test_non_power_of_two_tiles(gpu, mh, oracle, n, t):
    """Tile sides that are not powers of two (layout_test.cpp:23 allows them):
    the in-kernel Morton offsets take the division path, and t % 4 != 0 forces
    the element-wise epilogue edge path for every output."""
    rng = np.random.default_rng(n * 31 + t)
    for it, (q, op) in enumerate([(P16, OP_SUB), (97, OP_ADD), (P31, OP_SET), (P24, OP_SUB)]):
        r, k, c, corners = _random_views(rng, n)
        v = _views_from(oracle, n, t, r, k, c, corners)
        out, lhs, rhs = _fill(oracle, 2000 + it, n, q)
        got, _ = _run_gpu(mh, n, t, q, out, lhs, rhs, v, op)
        want = out.copy()
        oracle.mm_dense(n, t, q, want, lhs, rhs, v, op=op)
        assert np.array_equal(got, want), (n, t, q, op, v)


def test_reference_acceptance_instances(gpu, mh, oracle, reference):
    """acceptance_main.cpp:177-217 protocol: gen_problem draws, out += lhs*rhs,
    whole container equal to the reference's mm_oblivious, Counters equal."""
    for (n, t, q, seed, count) in [(64, 8, 2, 101, 40), (64, 8, 97, 102, 40), (256, 32, 2, 103, 12)]:
        g = oracle.rng(seed)
        for _ in range(count):
            out, lhs, rhs, _, v = oracle.gen_problem(g, n, t, q)
            got, ctr = _run_gpu(mh, n, t, q, out, lhs, rhs, v, OP_ADD)
            want = out.copy()
            ref = reference.mm_oblivious(n, t, q, want, lhs, rhs, v)
            assert np.array_equal(got, want)
            assert ctr.as_tuple() == ref.as_tuple()


def test_empty_problems_are_noops(gpu, mh, oracle):
    """multiply_test.cpp:187-193: empty problems leave the output, zero Counters."""
    n, t, q = 8, 4, 2
    out, lhs, rhs = _fill(oracle, 5, n, q)
    for dims in [(0, 4, 4), (4, 0, 4), (4, 4, 0)]:
        r, k, c = dims
        got, ctr = _run_gpu(mh, n, t, q, out, lhs, rhs, Views(0, 0, 0, r, k, c), OP_ADD)
        assert np.array_equal(got, out)
        assert ctr.as_tuple() == (0, 0, 0, 0, 0)


def test_validation_errors(gpu, mh):
    """multiply_test.cpp:165-185: the reference's exception classes."""
    two = mh.Modulus(2)
    A, B, C = (mh.Matrix(mh.Layout(8, 4), two) for _ in range(3))
    with pytest.raises(mh.LogicError):  # inner dimensions disagree
        mh.mm(mh.Problem(mh.Sub(A, 0, 4, 4), mh.Sub(B, 0, 4, 3), mh.Sub(C, 0, 4, 4)))
    with pytest.raises(mh.LogicError):  # shared container
        mh.mm(mh.Problem(mh.Sub(A, 0, 4, 4), mh.Sub(A, 0, 4, 4), mh.Sub(C, 0, 4, 4)))
    D = mh.Matrix(mh.Layout(8, 4), mh.Modulus(3))
    with pytest.raises(mh.LogicError):  # mixed moduli
        mh.mm(mh.Problem(mh.Sub(A, 0, 4, 4), mh.Sub(B, 0, 4, 4), mh.Sub(D, 0, 4, 4)))
    E = mh.Matrix(mh.Layout(8, 2), two)
    with pytest.raises(mh.LogicError):  # oblivious wants identical layouts
        mh.mm(mh.Problem(mh.Sub(A, 0, 4, 4), mh.Sub(B, 0, 4, 4), mh.Sub(E, 0, 4, 4)))
    with pytest.raises(mh.OutOfRange):
        mh.mm(mh.Problem(mh.Sub(A, 64, 1, 1), mh.Sub(B, 0, 1, 1), mh.Sub(C, 0, 1, 1)))
    with pytest.raises(mh.OutOfRange):
        mh.mm(mh.Problem(mh.Sub(A, 0, 9, 1), mh.Sub(B, 0, 9, 1), mh.Sub(C, 0, 1, 1)))
    with pytest.raises(mh.InvalidArgument):
        mh.mm(mh.Problem(mh.Sub(None, 0, 1, 1), mh.Sub(B, 0, 1, 1), mh.Sub(C, 0, 1, 1)))


def test_conversion_kernels_roundtrip(gpu, mh, oracle):
    """K1: from_row_major / to_row_major (matrix.hpp:44-67) vs the oracle codec."""
    for (n, t) in [(8, 4), (24, 3), (64, 8), (256, 64), (1024, 32)]:
        rng = np.random.default_rng(n + t)
        grid = rng.integers(0, 97, size=(n, n), dtype=np.uint32)
        m = mh.from_row_major(grid, t, mh.Modulus(97))
        assert np.array_equal(m.cells(), oracle.rowmajor_to_mh(n, t, grid))
        assert np.array_equal(mh.to_row_major(m), grid)
    with pytest.raises(mh.InvalidArgument):  # residue out of range (matrix.hpp:52-53)
        mh.from_row_major(np.full((8, 8), 97, np.uint32), 4, mh.Modulus(97))


# Residues whose signed limb digits are the extremes (+127 / -128 / -113 / +64 ...)
EXTREMES = {P16: (32639, 32640, P16 - 1, 0x807F, 1, 0xFEFF),
            P31: (1073741823, 1073741824, P31 - 1, 0x7F7F7F7F, 0x80808080 % P31)}


def _constant_case(mh, n, t, q, a, b, c0, k, op):
    """out (n x n, all c0) op= lhs (all a) * rhs (all b) over an r=c=n, inner k
    problem: every output cell must equal c0 +/- k*a*b mod q (closed form)."""
    lay, mod = mh.Layout(n, t), mh.Modulus(q)
    A = mh.Matrix(lay, mod).upload(np.full(n * n, c0, np.uint32))
    B = mh.Matrix(lay, mod).upload(np.full(n * n, a, np.uint32))
    Cm = mh.Matrix(lay, mod).upload(np.full(n * n, b, np.uint32))
    mh.mm(mh.Problem(mh.Sub(A, 0, n, n), mh.Sub(B, 0, n, k), mh.Sub(Cm, 0, k, n)), op)
    prod = (k * a * b) % q
    want = {OP_ADD: (c0 + prod) % q, OP_SUB: (c0 - prod) % q, OP_SET: prod}[op]
    got = A.cells()
    assert (got == want).all(), (q, a, b, op, int(got[0]), want)


@pytest.mark.parametrize("udig", ["0", "1"])
def test_adversarial_extreme_digits(gpu, mh, opts, udig):
    """Extreme-magnitude digits in every limb position (balanced s8 digits with
    MHG_OPT_DIGITS = 0, u8 digits by default), all three ops."""
    opts(mh.OPT_DIGITS, int(udig))
    for q, vals in EXTREMES.items():
        for a in vals:
            for b in vals[:3]:
                for op in (OP_ADD, OP_SUB, OP_SET):
                    _constant_case(mh, 1024, 64, q, a, b, q - 1, 1024, op)


def _extremes(q):
    """Residues whose signed representatives have extreme limb digits."""
    H = min((q - 1) // 2, 127 * 257)
    # (+ 0xFEFF: both u8 digits near 255 where it is a residue)
    return (H, q - H, q - 1, 1, (q + 1) // 2) + ((0xFEFF,) if q > 0xFEFF else ())


@pytest.mark.parametrize("udig", ["0", "1"])
@pytest.mark.parametrize("q,k", [(65287, 512), (65287, 640), (65519, 1024), (257, 1024), (65521, 4096),
                                 (65521, 8192)])
def test_single_reduction_fold_bound(gpu, mh, opts, q, k, udig):
    """Fold level 1 (single reduction, L=2) at the edge of its K bound:
    q = 65287 has 2^16 mod q = 249, so K = 512 is the largest chunk the host
    admits for s8 digits (K = 640 falls back to the per-class fold); the u8 levels'
    edges differ (mhg_fold_level_u8: 65521 on level 1 up to K = 4096); extreme
    digits, all ops."""
    opts(mh.OPT_DIGITS, int(udig))
    ex = _extremes(q)
    for a in ex:
        for b in ex[:2]:
            for op in (OP_ADD, OP_SUB, OP_SET):
                _constant_case(mh, max(1024, k), 64, q, a, b, q - 1, k, op)


@pytest.mark.parametrize("udig", ["0", "1"])
@pytest.mark.parametrize("level", ["2", "3"])
def test_forced_fold_levels(gpu, mh, opts, level, udig):
    """Fold levels 2 and 3 forced (MHG_OPT_MIN_FOLD_LEVEL) where level 1 would be chosen:
    the same exact results through every lean-fold arithmetic variant."""
    opts(mh.OPT_MIN_FOLD_LEVEL, int(level))
    opts(mh.OPT_DIGITS, int(udig))
    for q in (P16, 65287, 257):
        ex = _extremes(q)
        for a, b in [(ex[0], ex[0]), (ex[1], ex[0]), (ex[2], ex[4])]:
            for op in (OP_ADD, OP_SUB):
                _constant_case(mh, 1024, 64, q, a, b, q - 1, 1024, op)


@pytest.mark.slow
def test_single_reduction_fold_at_k8064(gpu, mh, opts):
    """p = 65521, s8 digits: the largest single-chunk K on fold level 1 (63 k-tiles)."""
    opts(mh.OPT_DIGITS, 0)
    ex = _extremes(P16)
    for a, b in [(ex[0], ex[0]), (ex[1], ex[0]), (ex[0], ex[1])]:
        _constant_case(mh, 8192, 64, P16, a, b, P16 - 1, 8064, OP_SUB)


@pytest.mark.slow
@pytest.mark.parametrize("udig", ["0", "1"])
def test_adversarial_int32_headroom(gpu, mh, opts, udig):
    """K = 32768 (cfg5's inner length) with extreme digits: the int32 class
    sums reach ~75% (q = 2^31-1) of the bound the planner sized chunks for (s8; u8
    digits take 2 / 4 chunks of 16,384 / 8,256)."""
    opts(mh.OPT_DIGITS, int(udig))
    for q in (P16, P31):
        for a, b in [(EXTREMES[q][0], EXTREMES[q][0]), (EXTREMES[q][1], EXTREMES[q][0])]:
            _constant_case(mh, 32768, 64, q, a, b, 1, 32768, OP_SUB)


def _u8_chunk_slices(q):
    """128-byte K slices per exact u8 chunk: (2^31 - 2^17) / (L * 255^2), the planner's
    bound for unsigned digits (mhg_planner.cpp gemm_geometry)."""
    L = mh_limbs(q)
    return ((1 << 31) - (1 << 17)) // (L * 255 * 255) // 128


def mh_limbs(q):
    L = 1
    while q > 256 ** L:
        L += 1
    return L


# Residues whose packed u8 digits are the largest the field allows: for p = 65521 the
# class-1 sum a0 b1 + a1 b0 peaks at 2 * 255 * 254 per k with 0xFEFF x 0xFEFF (99.6% of
# the 2 * 255^2 the chunk bound assumes); p - 1 = 0xFFF0 has the top digit 255.  For
# p = 2^31 - 1 the top digit is at most 127, so the widest classes peak at ~75%.
U8_MAX_DIGITS = {P16: (0xFEFF, P16 - 1, 0xFEFE), P31: (P31 - 1, 0x7EFFFFFF, 0x7FFFFEFF)}


def _device_constant_case(mh, n, t, q, a, b, c0, rows, k, cols, op, bufs):
    """Device-filled version of _constant_case for containers too large to stage on the
    host: out (rows x cols at the origin, all c0) op= lhs (rows x k, all a) * rhs (k x
    cols, all b).  The view is an aligned power-of-two block at (0, 0), so it is the flat
    range [0, rows*cols) of the output container; every view cell must equal
    c0 +/- k a b mod q and every other cell must still be c0."""
    import torch
    fo, fa, fb = bufs
    fo.fill_(int(c0))
    fa.fill_(int(a))
    fb.fill_(int(b))
    lay, mod = mh.Layout(n, t), mh.Modulus(q)
    A, B, Cm = (mh.Matrix.wrap(lay, mod, f.data_ptr(), owner=f) for f in bufs)
    mh.mm(mh.Problem(mh.Sub(A, 0, rows, cols), mh.Sub(B, 0, rows, k), mh.Sub(Cm, 0, k, cols)), op)
    prod = (k * a * b) % q
    want = {OP_ADD: (c0 + prod) % q, OP_SUB: (c0 - prod) % q, OP_SET: prod}[op]
    torch.cuda.synchronize()
    view = fo[:rows * cols]
    bad_view = int((view != int(want)).sum())
    bad_rest = int((fo[rows * cols:] != int(c0)).sum())
    assert bad_view == 0 and bad_rest == 0, (q, a, b, k, op, bad_view, bad_rest,
                                             int(view[0]) & 0xFFFFFFFF, want)


@pytest.mark.slow
@pytest.mark.parametrize("udig", [None, 0])
def test_u8_headroom_at_exact_chunk(gpu, mh, opts, udig):
    """SURVEY 8(c) 'adversarial max-limb inputs at the largest K per chunk', for the
    default u8 digits: K = one full exact chunk (p = 65521: 128 slices = 16,384, the
    north star's K; p = 2^31-1: 64 slices = 8,192) and one slice past it (two chunks),
    plus K = 16,384 for p = 2^31-1, with max-digit residues on both operands
    (for C -= A.B the lhs is p - x so that its packed digits are x's), C_old = p - 1,
    ADD / SUB / SET; digits as the planner picks them (udig None) and balanced s8."""
    import torch
    if udig is not None:
        opts(mh.OPT_DIGITS, udig)
    n, t, rows, cols = 32768, 64, 1024, 1024
    bufs = [torch.empty(n * n, dtype=torch.int32, device="cuda") for _ in range(3)]
    try:
        for q in (P16, P31):
            kc = _u8_chunk_slices(q) * 128
            ks = sorted({kc, kc + 128, 16384})
            vals = U8_MAX_DIGITS[q]
            for k in ks:
                for x, y in [(vals[0], vals[0]), (vals[0], vals[1]), (vals[1], vals[2])]:
                    for op in (OP_ADD, OP_SUB, OP_SET):
                        a = (q - x) % q if op == OP_SUB else x  # packed lhs digits = x's
                        _device_constant_case(mh, n, t, q, a, y, q - 1, rows, k, cols, op, bufs)
    finally:
        del bufs
        torch.cuda.empty_cache()


def test_u8_chunk_bound_is_the_planner_bound(gpu, mh):
    """The K chunks the headroom test targets are exactly the planner's: one chunk at
    K = 16,384 (p = 65521) / 8,192 (p = 2^31-1), two one slice later."""
    def chunks(q, k):
        lay, mod = mh.Layout(16384 * 2, 64), mh.Modulus(q)
        A, B, C = (mh.Matrix(lay, mod) for _ in range(3))
        return mh.Plan(mh.Problem(mh.Sub(A, 0, 128, 128), mh.Sub(B, 0, 128, k),
                                  mh.Sub(C, 0, k, 128)), mh.OP_SUB).info()["k_chunks"]
    assert _u8_chunk_slices(P16) == 128 and _u8_chunk_slices(P31) == 64
    for q in (P16, P31):
        kc = _u8_chunk_slices(q) * 128
        assert chunks(q, kc) == 1 and chunks(q, kc + 128) == 2


@pytest.mark.slow
def test_north_star_u8_equals_s8(gpu, mh, opts):
    """The bench workload (n = 16384, p = 65521, C -= A.B, uniform residues) with u8
    and with balanced s8 digits: byte-identical output containers."""
    import torch
    n, t, q = 16384, 64, P16
    g = torch.Generator(device="cuda").manual_seed(2024)
    src = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda", generator=g) for _ in range(3)]
    outs = []
    for digits in (1, 0):
        opts(mh.OPT_DIGITS, digits)
        fo = src[0].clone()
        lay, mod = mh.Layout(n, t), mh.Modulus(q)
        A = mh.Matrix.wrap(lay, mod, fo.data_ptr(), owner=fo)
        B = mh.Matrix.wrap(lay, mod, src[1].data_ptr(), owner=src[1])
        C = mh.Matrix.wrap(lay, mod, src[2].data_ptr(), owner=src[2])
        plan = mh.Plan(mh.Problem(mh.Sub(A, 0, n, n), mh.Sub(B, 0, n, n), mh.Sub(C, 0, n, n)), OP_SUB)
        assert plan.info()["digits"] == ("u8" if digits else "s8")
        plan.run()
        torch.cuda.synchronize()
        outs.append(fo)
        del plan
    assert torch.equal(outs[0], outs[1])
    assert not torch.equal(outs[0], src[0])


@pytest.mark.parametrize("udig", ["0", "1"])
def test_k_chunking(gpu, mh, oracle, opts, udig):
    """Multi-chunk accumulation (each exact int32 K-chunk drained and folded into
    the output before the next): forced to 2 K-slices per chunk so small
    problems take the path n >= 65536 would take for q = 2^31-1."""
    opts(mh.OPT_MAX_KCHUNK, 2)
    opts(mh.OPT_DIGITS, int(udig))
    rng = np.random.default_rng(77)
    for q in (P16, P31):
        for op in (OP_ADD, OP_SUB, OP_SET):
            n, t = 1024, 64
            r, k, c, corners = _random_views(rng, n, r=300, k=1000, c=200)
            v = _views_from(oracle, n, t, r, k, c, corners)
            out, lhs, rhs = _fill(oracle, 9 + op, n, q)
            got, _ = _run_gpu(mh, n, t, q, out, lhs, rhs, v, op)
            want = out.copy()
            oracle.mm_dense(n, t, q, want, lhs, rhs, v, op=op)
            assert np.array_equal(got, want), (q, op)


@pytest.mark.slow
def test_cfg2_full_container(gpu, mh, oracle):
    """BASELINE cfg2: n=4096, t=64, p=65521, C -= A*B, C uniform: whole container."""
    n, t, q = 4096, 64, P16
    out, lhs, rhs = _fill(oracle, 0, n, q)
    v = Views(0, 0, 0, n, n, n)
    got, _ = _run_gpu(mh, n, t, q, out, lhs, rhs, v, OP_SUB)
    want = out.copy()
    oracle.mm_dense(n, t, q, want, lhs, rhs, v, op=OP_SUB)
    assert np.array_equal(got, want)


@pytest.mark.slow
def test_cfg3_misaligned_schur_update(gpu, mh, oracle):
    """BASELINE cfg3: C(6144x5120) -= A(6144x2048) B(2048x5120) in 8192^2 parents
    at (96,160), t=64 -- exercises the alignment/containment decomposition."""
    n, t, q = 8192, 64, P16
    out, lhs, rhs = _fill(oracle, 3, n, q)
    v = Views(oracle.encode(n, t, 96, 160), oracle.encode(n, t, 96, 160),
              oracle.encode(n, t, 96, 160), 6144, 2048, 5120)
    got, ctr = _run_gpu(mh, n, t, q, out, lhs, rhs, v, OP_SUB)
    assert ctr.base_case_calls == 97 * 33 * 81  # 259,281 leaves
    want = out.copy()
    oracle.mm_dense(n, t, q, want, lhs, rhs, v, op=OP_SUB)
    assert np.array_equal(got, want)


def _reference_tiles(reference, oracle, n, t, q, out, lhs, rhs, got, op, tiles):
    """Recompute 64 x 64 output tiles with the REFERENCE's own mm_oblivious
    (oracle/_ref: the reference headers compiled in place) on a copy of the
    original C -- the tile's row panel of A and column panel of B as views -- and
    compare those cells with the GPU result (full views only)."""
    ref_out = out.copy()
    for (r0, c0) in tiles:
        tv = Views(oracle.encode(n, t, r0, c0), oracle.encode(n, t, r0, 0),
                   oracle.encode(n, t, 0, c0), 64, n, 64)
        reference.mm(2, n, t, q, ref_out, lhs, rhs, tv, op=op)
        idx = [oracle.encode(n, t, r0 + a, c0 + b) for a in range(64) for b in range(64)]
        assert np.array_equal(got[idx], ref_out[idx]), (r0, c0)


def _sampled_tiles(oracle, n, t, q, out, lhs, rhs, got, v, op, tiles):
    for (r0, c0) in tiles:
        nr, nc = min(64, v.rows - r0), min(64, v.cols - c0)
        want = oracle.mm_dense_block(n, t, q, out, lhs, rhs, v, r0, nr, c0, nc, op=op)
        oi, oj = oracle.extract(n, t, v.out_origin)
        for a in range(nr):
            idx = [oracle.encode(n, t, oi + r0 + a, oj + c0 + b) for b in range(nc)]
            assert np.array_equal(got[idx], want[a]), (r0, c0, a)


@pytest.mark.slow
def test_cfg4_large_prime(gpu, mh, oracle):
    """BASELINE cfg4: n=8192, t=64, p=2^31-1, C = A*B: Freivalds + sampled tiles."""
    n, t, q = 8192, 64, P31
    out, lhs, rhs = _fill(oracle, 4, n, q)
    v = Views(0, 0, 0, n, n, n)
    got, _ = _run_gpu(mh, n, t, q, out, lhs, rhs, v, OP_SET)
    assert oracle.freivalds(n, t, q, out, lhs, rhs, got, v, op=OP_SET, rounds=2)
    h = n // 2
    _sampled_tiles(oracle, n, t, q, out, lhs, rhs, got, v, OP_SET,
                   [(0, 0), (0, h), (h, 0), (h, h), (n - 64, n - 64), (h - 32, h - 32)])
    if reference_available():
        from oracle.binding import Reference
        _reference_tiles(Reference(), oracle, n, t, q, out, lhs, rhs, got, OP_SET,
                         [(0, 64), (h, h - 64)])
    bad = got.copy()
    bad[12345] = (bad[12345] + 1) % q
    assert not oracle.freivalds(n, t, q, out, lhs, rhs, bad, v, op=OP_SET, rounds=1)


@pytest.mark.slow
def test_north_star_size(gpu, mh, oracle):
    """n=16384, t=64, p=65521, C -= A*B (the bench workload): Freivalds over the
    whole result + tiles in every top-level Morton quadrant, edges, corners."""
    n, t, q = 16384, 64, P16
    out, lhs, rhs = _fill(oracle, 0, n, q)
    v = Views(0, 0, 0, n, n, n)
    got, ctr = _run_gpu(mh, n, t, q, out, lhs, rhs, v, OP_SUB)
    assert ctr.scalar_macs == n ** 3
    assert oracle.freivalds(n, t, q, out, lhs, rhs, got, v, op=OP_SUB, rounds=2)
    h = n // 2
    _sampled_tiles(oracle, n, t, q, out, lhs, rhs, got, v, OP_SUB,
                   [(0, 0), (0, h), (h, 0), (h, h), (0, n - 64), (n - 64, 0), (n - 64, n - 64)])


@pytest.mark.slow
def test_north_star_against_reference_tiles(gpu, mh, oracle, reference):
    """The bench workload checked against the reference implementation itself:
    tiles in all four top-level Morton quadrants recomputed by the reference's
    mm_oblivious (C -= A*B through its Sub-view API) equal the GPU result."""
    n, t, q = 16384, 64, P16
    out, lhs, rhs = _fill(oracle, 0, n, q)
    got, _ = _run_gpu(mh, n, t, q, out, lhs, rhs, Views(0, 0, 0, n, n, n), OP_SUB)
    h = n // 2
    _reference_tiles(reference, oracle, n, t, q, out, lhs, rhs, got, OP_SUB,
                     [(0, 0), (64, h + 128), (h, 192), (n - 64, n - 64)])


def test_alias_mode_same_parent(gpu, mh, oracle):
    """TU Schur update on views of ONE parent: rejected by default (the
    reference's rule), exact with allow_alias (snapshot semantics), including
    overlapping views."""
    n, t, q = 256, 32, P16
    (cells,) = _fill(oracle, 21, n, q)[:1]
    lay, mod = mh.Layout(n, t), mh.Modulus(q)
    M = mh.Matrix(lay, mod).upload(cells)
    prob = mh.Problem(mh.Sub(M, mh.encode(lay, 100, 100), 156, 156),
                      mh.Sub(M, mh.encode(lay, 100, 37), 156, 63),
                      mh.Sub(M, mh.encode(lay, 37, 100), 63, 156))
    with pytest.raises(mh.LogicError):
        mh.mm(prob)
    for views, op in [((100, 100, 100, 37, 37, 100, 156, 63, 156), OP_SUB),
                      ((0, 0, 10, 5, 20, 30, 200, 150, 180), OP_ADD)]:  # overlapping
        oi, oj, li, lj, ri, rj, r, k, c = views
        M.upload(cells)
        prob = mh.Problem(mh.Sub(M, mh.encode(lay, oi, oj), r, c), mh.Sub(M, mh.encode(lay, li, lj), r, k),
                          mh.Sub(M, mh.encode(lay, ri, rj), k, c))
        mh.mm(prob, op, allow_alias=True)
        got = M.cells()
        want = cells.copy()
        v = Views(oracle.encode(n, t, oi, oj), oracle.encode(n, t, li, lj), oracle.encode(n, t, ri, rj),
                  r, k, c)
        oracle.mm_dense(n, t, q, want, cells.copy(), cells.copy(), v, op=op)
        assert np.array_equal(got, want), views


def test_tu_schur_sweep(gpu, mh, oracle):
    """Right-looking elimination update sweep on one parent, misaligned panel
    width (96 vs t=64), every step a graph-replayed aliased plan."""
    from paper_1705_04807_b200.tu import schur_plans, schur_sweep
    n, t, q, block = 1024, 64, P16, 96
    (cells,) = _fill(oracle, 22, n, q)[:1]
    lay, mod = mh.Layout(n, t), mh.Modulus(q)
    M = mh.Matrix(lay, mod).upload(cells)
    plans = schur_plans(M, block)
    macs = schur_sweep(M, block, plans=plans)
    got = M.cells()
    want = cells.copy()
    k0 = 0
    while k0 + block < n:
        k1, rest = k0 + block, n - k0 - block
        v = Views(oracle.encode(n, t, k1, k1), oracle.encode(n, t, k1, k0), oracle.encode(n, t, k0, k1),
                  rest, block, rest)
        oracle.mm_dense(n, t, q, want, want.copy(), want.copy(), v, op=OP_SUB)
        k0 = k1
    assert np.array_equal(got, want)
    assert macs == sum(((n - k) ** 2) * block for k in range(block, n, block))


@pytest.mark.filterwarnings("ignore:The CUDA Graph is empty")
def test_tu_sweep_graph(gpu, mh, oracle):
    """tu.SweepGraph: the whole aliased sweep captured into one CUDA graph; two replays equal
    two oracle sweeps (every step reads the previous step's output from the parent)."""
    import torch
    from paper_1705_04807_b200.tu import SweepGraph
    n, t, q, block = 512, 32, P16, 128
    (cells,) = _fill(oracle, 23, n, q)[:1]
    lay, mod = mh.Layout(n, t), mh.Modulus(q)
    M = mh.Matrix(lay, mod).upload(cells)
    sg = SweepGraph(M, block)
    want = cells.copy()
    for rep in range(2):
        macs = sg.replay()
        k0 = 0
        while k0 + block < n:
            k1, rest = k0 + block, n - k0 - block
            v = Views(oracle.encode(n, t, k1, k1), oracle.encode(n, t, k1, k0), oracle.encode(n, t, k0, k1),
                      rest, block, rest)
            oracle.mm_dense(n, t, q, want, want.copy(), want.copy(), v, op=OP_SUB)
            k0 = k1
        torch.cuda.synchronize()
        assert np.array_equal(M.cells(), want), rep
    assert macs == sum(((n - k) ** 2) * block for k in range(block, n, block))
    # the same sequence on a side stream; degenerate sequences
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    sg.replay(side)
    side.synchronize()
    assert not np.array_equal(M.cells(), want)  # a third sweep ran
    assert SweepGraph(M, n).replay() == 0       # block >= n: no steps
    with pytest.raises(mh.InvalidArgument):
        mh.Sweep([])
    pl = sg.plans[0]
    pl.set_profiling(True)
    with pytest.raises(mh.Unsupported):
        mh.Sweep([pl])
    pl.set_profiling(False)
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    with pytest.raises(mh.Unsupported):       # a capturing stream takes the plans, not the sweep
        with torch.cuda.graph(g, stream=cap):
            sg.replay(cap)


@pytest.mark.parametrize("kernel", [1, 2])
def test_both_gemm_kernels(gpu, mh, oracle, opts, kernel):
    """The single-CTA (k_gemm) and CTA-pair (k_gemm2, cta_group::2) kernels
    (MHG_OPT_GEMM_KERNEL = 1 / 2) on ragged views, every limb count, all ops, forced
    K-chunking."""
    opts(mh.OPT_GEMM_KERNEL, kernel)
    rng = np.random.default_rng(5)
    for q in (97, P16, P24, P31):
        for op in (OP_ADD, OP_SUB, OP_SET):
            n = 512
            t = int(rng.choice([16, 32, 64]))
            r, k, c, corners = _random_views(rng, n)
            v = _views_from(oracle, n, t, r, k, c, corners)
            out, lhs, rhs = _fill(oracle, 40 + op, n, q)
            if op == OP_SUB:
                opts(mh.OPT_MAX_KCHUNK, 1)
            got, _ = _run_gpu(mh, n, t, q, out, lhs, rhs, v, op)
            opts(mh.OPT_MAX_KCHUNK, 0)
            want = out.copy()
            oracle.mm_dense(n, t, q, want, lhs, rhs, v, op=op)
            assert np.array_equal(got, want), (kernel, q, op, t, v)


def test_edge_shapes(gpu, mh, oracle):
    """Degenerate and boundary shapes: 1x1 containers, t = 1, t = n, views
    that touch every container edge, single rows / columns / inner length 1,
    non-power-of-two tiles."""
    cases = [
        (1, 1, 97, (0, 0, 0, 0, 0, 0), 1, 1, 1),
        (2, 1, 97, (0, 0, 0, 0, 0, 0), 2, 2, 2),
        (64, 64, 65521, (0, 0, 0, 0, 0, 0), 64, 64, 64),       # one tile
        (128, 1, 65521, (3, 5, 7, 9, 11, 13), 100, 90, 80),    # t = 1 (pure Z order)
        (96, 3, 257, (0, 1, 2, 3, 3, 5), 91, 93, 90),          # non-pow2 tile side
        (256, 64, P31, (255, 0, 0, 255, 0, 0), 1, 1, 256),     # single row, inner 1
        (256, 64, P31, (0, 255, 0, 0, 0, 255), 256, 256, 1),   # single column
        (256, 32, P16, (1, 1, 1, 1, 1, 1), 255, 255, 255),     # touches the far edges
    ]
    for (n, t, q, corners, r, k, c) in cases:
        v = _views_from(oracle, n, t, r, k, c, corners)
        out, lhs, rhs = _fill(oracle, n + t, n, q)
        for op in (OP_ADD, OP_SUB, OP_SET):
            got, _ = _run_gpu(mh, n, t, q, out, lhs, rhs, v, op)
            want = out.copy()
            oracle.mm_dense(n, t, q, want, lhs, rhs, v, op=op)
            assert np.array_equal(got, want), (n, t, q, corners, r, k, c, op)


def test_plan_graph_replay_matches_direct(gpu, mh, oracle):
    """A plan replayed as a CUDA graph (several runs) equals repeated direct
    calls, and its Counters equal the direct call's."""
    n, t, q = 512, 32, P16
    out, lhs, rhs = _fill(oracle, 77, n, q)
    v = _views_from(oracle, n, t, 300, 200, 250, (10, 20, 30, 40, 50, 60))
    A, B, Cm = _containers(mh, n, t, q, (out, lhs, rhs))
    prob = mh.Problem(mh.Sub(A, v.out_origin, v.rows, v.cols), mh.Sub(B, v.lhs_origin, v.rows, v.inner),
                      mh.Sub(Cm, v.rhs_origin, v.inner, v.cols))
    plan = mh.Plan(prob, mh.OP_SUB)
    for _ in range(3):
        plan.run()
    got = A.cells()
    want = out.copy()
    for _ in range(3):
        oracle.mm_dense(n, t, q, want, lhs, rhs, v, op=OP_SUB)
    assert np.array_equal(got, want)
    assert plan.counters().as_tuple() == mh.counters_oblivious(prob).as_tuple()
    assert plan.info()["launches"] == 2  # k_pack_pair + k_gemm


@pytest.mark.parametrize("kernel", [1, 2])
def test_guard_bands(gpu, mh, oracle, opts, kernel):
    """Out-of-bounds detector (compute-sanitizer is unavailable on this pool):
    each container is wrapped in the middle of a larger device buffer whose
    guard zones hold a sentinel; after multiplies with ragged views, every
    guard word is intact and the result equals the oracle."""
    import torch
    opts(mh.OPT_GEMM_KERNEL, kernel)
    n, t, guard = 256, 32, 1 << 16
    sentinel = 0x5A5A5A5A
    for q in (97, P16, P31):
        lay, mod = mh.Layout(n, t), mh.Modulus(q)
        cells = _fill(oracle, q % 1000, n, q)
        bufs, mats = [], []
        for c in cells:
            b = torch.full((n * n + 2 * guard,), sentinel, dtype=torch.int64, device="cuda").to(torch.int32)
            b[guard:guard + n * n] = torch.from_numpy(c.view(np.int32)).cuda()
            bufs.append(b)
            mats.append(mh.Matrix.wrap(lay, mod, b[guard:].data_ptr(), owner=b))
        v = _views_from(oracle, n, t, 250, 131, 7, (5, 249, 1, 3, 120, 240))
        for op in (OP_SUB, OP_SET, OP_ADD):
            mh.mm(mh.Problem(mh.Sub(mats[0], v.out_origin, v.rows, v.cols),
                             mh.Sub(mats[1], v.lhs_origin, v.rows, v.inner),
                             mh.Sub(mats[2], v.rhs_origin, v.inner, v.cols)), op)
            oracle.mm_dense(n, t, q, cells[0], cells[1], cells[2], v, op=op)
        torch.cuda.synchronize()
        for b in bufs:
            h = b.cpu().numpy().view(np.uint32)
            assert (h[:guard] == sentinel).all() and (h[guard + n * n:] == sentinel).all()
        assert np.array_equal(bufs[0][guard:guard + n * n].cpu().numpy().view(np.uint32), cells[0])
        assert np.array_equal(bufs[1][guard:guard + n * n].cpu().numpy().view(np.uint32), cells[1])


def test_reference_golden_cases(gpu, mh, oracle):
    """tests/golden/cases.json (generated by running the reference library,
    tests/golden/make_golden.py): for every case the GPU's whole output
    container hashes to the reference's SHA-256 and the Counters match."""
    import hashlib
    import json
    import os
    cases = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cases.json")))
    assert len(cases) >= 60
    for c in cases:
        n, t, q = c["n"], c["t"], c["q"]
        g = oracle.rng(c["seed"])
        for _ in range(c["draw"]):
            oracle.gen_problem(g, n, t, q)
        out, lhs, rhs, _, v = oracle.gen_problem(g, n, t, q)
        assert [v.out_origin, v.lhs_origin, v.rhs_origin, v.rows, v.inner, v.cols] == c["views"]
        got, ctr = _run_gpu(mh, n, t, q, out, lhs, rhs, v, c["op"])
        assert hashlib.sha256(got.tobytes()).hexdigest() == c["out_sha256"], c
        assert list(ctr.as_tuple()) == c["counters"], c


@pytest.mark.slow
def test_cfg5_box_scale(gpu, mh, oracle):
    """BASELINE cfg5 shape on one GPU: n=32768, t=64, p=65521, C -= A*B (K=32768
    in a single exact int32 chunk): Freivalds over the whole result + tiles in
    the four top-level quadrants and the far corner."""
    n, t, q = 32768, 64, P16
    out, lhs, rhs = _fill(oracle, 5, n, q)
    v = Views(0, 0, 0, n, n, n)
    got, ctr = _run_gpu(mh, n, t, q, out, lhs, rhs, v, OP_SUB)
    assert ctr.base_case_calls == 512 ** 3
    assert oracle.freivalds(n, t, q, out, lhs, rhs, got, v, op=OP_SUB, rounds=1)
    h = n // 2
    _sampled_tiles(oracle, n, t, q, out, lhs, rhs, got, v, OP_SUB,
                   [(0, 0), (0, h), (h, 0), (h, h), (n - 64, n - 64)])


@pytest.mark.slow
def test_two_exact_chunks_at_scale(gpu, mh, oracle):
    """n = 65536: K = 65536 exceeds the exact int32 chunk for p = 65521
    (k_max = 65532), so the GEMM really drains and folds two K-chunks per tile.
    Whole-result Freivalds check (inputs from numpy; 16 GiB per container)."""
    n, t, q = 65536, 64, P16
    L, H, kmax = mh.limb_params(q)
    assert n > kmax
    rng = np.random.default_rng(65536)
    out, lhs, rhs = (rng.integers(0, q, n * n, dtype=np.uint32) for _ in range(3))
    v = Views(0, 0, 0, n, n, n)
    got, ctr = _run_gpu(mh, n, t, q, out, lhs, rhs, v, OP_SUB)
    assert ctr.scalar_macs == n ** 3
    assert oracle.freivalds(n, t, q, out, lhs, rhs, got, v, op=OP_SUB, rounds=1)


def test_concurrent_calls_on_streams(gpu, mh, oracle):
    """Concurrent one-shot multiplies and plans from several host threads on their
    own streams (disjoint outputs -- the reference's concurrency contract,
    multiply.hpp:25-29): the shared one-shot workspace is ordered by events, plans
    own theirs; every result must equal the oracle's."""
    import threading

    import torch

    n, t, q = 256, 32, P16
    jobs = []
    for w in range(3):
        rng = np.random.default_rng(900 + w)
        out, lhs, rhs = _fill(oracle, 900 + w, n, q)
        A, B, Cm = _containers(mh, n, t, q, (out, lhs, rhs))
        seq = []
        want = out.copy()
        for it in range(4):
            r, k, c, corners = _random_views(rng, n)
            v = _views_from(oracle, n, t, r, k, c, corners)
            seq.append(v)
            oracle.mm_dense(n, t, q, want, lhs, rhs, v, op=OP_SUB)
        jobs.append((A, B, Cm, seq, want))
    errors = []

    def worker(job, use_plan):
        try:
            A, B, Cm, seq, _ = job
            s = torch.cuda.Stream()
            for v in seq:
                prob = mh.Problem(mh.Sub(A, v.out_origin, v.rows, v.cols),
                                  mh.Sub(B, v.lhs_origin, v.rows, v.inner),
                                  mh.Sub(Cm, v.rhs_origin, v.inner, v.cols))
                if use_plan:
                    mh.Plan(prob, mh.OP_SUB).run(s)
                else:
                    mh.mm(prob, mh.OP_SUB, stream=s)
            s.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(j, i == 2)) for i, j in enumerate(jobs)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    torch.cuda.synchronize()
    assert not errors, errors
    for A, _, _, _, want in jobs:
        assert np.array_equal(A.cells(), want)


def test_split_plan_execution(gpu, mh, oracle):
    """mhg_plan_pack / pack_buffer / gemm (the packed multi-GPU exchange): packing
    both operands then running the GEMM equals the oracle; a packed operand copied
    into another plan of the same geometry is consumed as-is; bad arguments raise."""
    import torch

    n, t, q = 256, 32, P16
    out, lhs, rhs = _fill(oracle, 1700, n, q)
    A, B, Cm = _containers(mh, n, t, q, (out, lhs, rhs))
    v = _views_from(oracle, n, t, 200, 150, 170, [30, 40, 20, 60, 50, 70])
    prob = mh.Problem(mh.Sub(A, v.out_origin, v.rows, v.cols), mh.Sub(B, v.lhs_origin, v.rows, v.inner),
                      mh.Sub(Cm, v.rhs_origin, v.inner, v.cols))
    pl = mh.Plan(prob, mh.OP_SUB)
    pl.pack(0)
    pl.pack(1)
    pl.gemm()
    torch.cuda.synchronize()
    want = out.copy()
    oracle.mm_dense(n, t, q, want, lhs, rhs, v, op=OP_SUB)
    assert np.array_equal(A.cells(), want)
    # a second plan over the same shapes on other containers, fed the first plan's packs
    A2, B2, C2 = _containers(mh, n, t, q, (out, np.zeros_like(lhs), np.zeros_like(rhs)))
    pl2 = mh.Plan(mh.Problem(mh.Sub(A2, v.out_origin, v.rows, v.cols),
                             mh.Sub(B2, v.lhs_origin, v.rows, v.inner),
                             mh.Sub(C2, v.rhs_origin, v.inner, v.cols)), mh.OP_SUB)
    for which in (0, 1):
        dst, src = pl2.pack_buffer(which), pl.pack_buffer(which)
        assert dst.numel() == src.numel() > 0
        dst.copy_(src)
    pl2.gemm()
    torch.cuda.synchronize()
    assert np.array_equal(A2.cells(), want)
    with pytest.raises(mh.InvalidArgument):
        pl.pack(2)


@pytest.mark.parametrize("P,op", [(2, "sub"), (4, "set"), (8, "add")])
def test_dist_segment_plans_cover_the_multiply(gpu, mh, oracle, P, op):
    """mhg_dist_plan_create (the C ABI's multi-GPU partition): every rank's K-segment plans,
    run one after another on ONE device over full containers, make exactly the whole
    multiply (SET overwrites with segment 0 and accumulates the rest) and their MACs sum
    to n^3; the SET form rejects nothing the plain plan accepts."""
    import torch

    n, t, q = 512, 32, P16
    out, lhs, rhs = _fill(oracle, 4200 + P, n, q)
    A, B, Cm = _containers(mh, n, t, q, (out, lhs, rhs))
    code = {"add": mh.OP_ADD, "sub": mh.OP_SUB, "set": mh.OP_SET}[op]
    macs = 0
    for r in range(P):
        segs = mh.dist_segments(P, r, n, t)
        blk = mh.dist_block(P, r, n, t)
        assert sum(g.k1 - g.k0 for g in segs) == n
        for g in segs:
            pl = mh.Plan.for_segment(A, B, Cm, code, P, r, g.index)
            assert pl.counters().scalar_macs == blk.rows * blk.cols * (g.k1 - g.k0)
            macs += pl.counters().scalar_macs
            pl.run()
    torch.cuda.synchronize()
    assert macs == n ** 3
    want = out.copy()
    full = _views_from(oracle, n, t, n, n, n, [0] * 6)
    oracle.mm_dense(n, t, q, want, lhs, rhs, full, op={"add": OP_ADD, "sub": OP_SUB, "set": OP_SET}[op])
    assert np.array_equal(A.cells(), want)
    with pytest.raises(mh.OutOfRange):
        mh.Plan.for_segment(A, B, Cm, code, P, P, 0)
    with pytest.raises(mh.OutOfRange):
        mh.Plan.for_segment(A, B, Cm, code, P, 0, 64)


@pytest.mark.parametrize("n,t,q,bad", [
    (4096, 64, P16, ()),                   # 4 staging chunks, all cells on the 16-bit wire
    (6144, 96, P16, ()),                   # non-pow2 tile, partial last chunk
    (2049, 2049, P16, ()),                 # odd cell count: widen tail
    (6144, 96, P16, (20_000_000,)),        # a cell >= 2^16 in chunk 4: the rest as 4-byte cells
    (4096, 64, P16, (5, 16_777_215)),      # ... in the first chunk: all 4-byte cells
    (2048, 64, 65537, ()),                 # q > 2^16: plain copy
])
def test_upload_wire16_equals_plain_copy(gpu, mh, n, t, q, bad):
    """mhg_matrix_upload's 16-bit wire leaves the container byte-identical to a
    plain copy of the host buffer (Matrix::cells(), matrix.hpp:27-28); from the
    first chunk holding a wide cell on, the buffer travels as 4-byte cells."""
    rng = np.random.default_rng(n + sum(bad))
    cells = rng.integers(0, min(q, 65536), size=n * n, dtype=np.uint32)
    for b in bad:
        cells[b] = 0x12345678 + b
    m = mh.Matrix(mh.Layout(n, t), mh.Modulus(q))
    m.upload(cells)
    assert np.array_equal(m.cells(), cells)
    chunk, total = 1 << 22, n * n  # the wire's staging chunk (mhg_wire.cpp)
    if q > 65536:
        assert m.upload_bytes == 4 * total
    else:
        narrow = min(bad) // chunk * chunk if bad else total
        assert m.upload_bytes == 2 * narrow + 4 * (total - narrow)
    # re-upload over stale contents, on a side stream, from pinned memory
    import torch
    s = torch.cuda.Stream()
    h = torch.from_numpy(cells[::-1].copy().view(np.int32)).pin_memory()
    mh._check(mh.lib().mhg_matrix_upload(m.handle, h.data_ptr(), s.cuda_stream))
    torch.cuda.synchronize()
    assert np.array_equal(m.cells(), cells[::-1])


def test_upload_range(gpu, mh):
    """mhg_matrix_upload_range: one flat cell range (a rank's Morton slice) from a
    host buffer holding exactly those cells, on the 16-bit wire (>= 4M cells) or
    as a plain copy; the rest of the container is untouched; bounds checked."""
    n, t, q = 4096, 64, P16
    rng = np.random.default_rng(3)
    base = rng.integers(0, q, size=n * n, dtype=np.uint32)
    m = mh.Matrix(mh.Layout(n, t), mh.Modulus(q)).upload(base)
    want = base.copy()
    for off, cnt in [(12345, 5_000_000), (n * n - 4_194_304, 4_194_304), (7, 1000), (0, 0)]:
        part = rng.integers(0, q, size=cnt, dtype=np.uint32)
        mh._check(mh.lib().mhg_matrix_upload_range(m.handle, part.ctypes.data, off, cnt, None))
        want[off:off + cnt] = part
        assert np.array_equal(m.cells(), want), (off, cnt)
        assert m.upload_bytes == (2 if cnt >= 1 << 22 else 4) * cnt or cnt == 0
    with pytest.raises(mh.OutOfRange):
        mh._check(mh.lib().mhg_matrix_upload_range(m.handle, base.ctypes.data, n * n - 10, 11, None))


def test_concurrent_uploads_from_threads(gpu, mh):
    """Uploads on the 16-bit wire from several host threads at once (own streams,
    distinct containers, pinned and pageable sources, full and range uploads):
    they share one narrowing pool and staging ring and must each land exactly."""
    import threading

    import torch

    n, t, q = 4096, 64, P16  # halves of 8M cells: both range uploads on the wire
    rng = np.random.default_rng(44)
    srcs = [rng.integers(0, q, size=n * n, dtype=np.uint32) for _ in range(4)]
    mats = [mh.Matrix(mh.Layout(n, t), mh.Modulus(q)) for _ in range(4)]
    errors = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            src = srcs[i]
            for rep in range(3):
                if i % 2:
                    h = torch.from_numpy(src.view(np.int32)).pin_memory()
                    mh._check(mh.lib().mhg_matrix_upload(mats[i].handle, h.data_ptr(), s.cuda_stream))
                    s.synchronize()
                else:
                    half = n * n // 2 + 8 * rep + 1
                    mh._check(mh.lib().mhg_matrix_upload_range(mats[i].handle, src.ctypes.data, 0,
                                                               half, s.cuda_stream))
                    mh._check(mh.lib().mhg_matrix_upload_range(
                        mats[i].handle, src[half:].ctypes.data, half, n * n - half, s.cuda_stream))
                    s.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for m, src in zip(mats, srcs):
        assert np.array_equal(m.cells(), src)
        assert m.upload_bytes <= 2 * n * n  # the last (range or full) upload was narrow


@pytest.mark.parametrize("conv", [0, 1, 2])
def test_conversion_kernel_variants(gpu, mh, oracle, opts, conv):
    """K1 on device buffers through the C ABI: the TMA kernel (MHG_OPT_CONV_KERNEL = 0,
    default; units of R rows x t columns, R < t from t = 128 on), the Morton-order
    LDG/STG kernel (1) and the row-order one (2), for t = 4 ... 256 and a
    non-power-of-two tile (fallback); round trip exact; an out-of-range residue in the
    last unit is reported; misaligned row buffers fall back."""
    import torch
    opts(mh.OPT_CONV_KERNEL, conv)
    lib = mh.lib()
    for (n, t) in [(8, 4), (64, 8), (1024, 32), (2048, 64), (2048, 128), (4096, 256), (96, 6)]:
        q = 65521
        rng = np.random.default_rng(n + t)
        grid = rng.integers(0, q, size=(n, n), dtype=np.uint32)
        m = mh.Matrix(mh.Layout(n, t), mh.Modulus(q))
        rm = torch.from_numpy(grid.reshape(-1).view(np.int32)).cuda()
        assert lib.mhg_rowmajor_to_mh(m.handle, rm.data_ptr(), None) == 0
        assert np.array_equal(m.cells(), oracle.rowmajor_to_mh(n, t, grid)), (n, t)
        back = torch.zeros_like(rm)
        assert lib.mhg_mh_to_rowmajor(m.handle, back.data_ptr(), None) == 0
        torch.cuda.synchronize()
        assert np.array_equal(back.cpu().numpy().view(np.uint32).reshape(n, n), grid), (n, t)
        bad = rm.clone()
        bad[-1] = q
        assert lib.mhg_rowmajor_to_mh(m.handle, bad.data_ptr(), None) == 1, (n, t)
    # misaligned row-major buffer (4-byte offset): LDG/STG fallback, same result
    n, t = 1024, 64
    grid = np.random.default_rng(1).integers(0, 97, size=(n, n), dtype=np.uint32)
    m = mh.Matrix(mh.Layout(n, t), mh.Modulus(97))
    buf = torch.zeros(n * n + 1, dtype=torch.int32, device="cuda")
    buf[1:] = torch.from_numpy(grid.reshape(-1).view(np.int32)).cuda()
    assert lib.mhg_rowmajor_to_mh(m.handle, buf.data_ptr() + 4, None) == 0
    assert np.array_equal(m.cells(), oracle.rowmajor_to_mh(n, t, grid))


def test_planner_kernel_policy(gpu, mh, opts):
    """mhg_plan_variant: u8 digits by default (s8 with MHG_OPT_DIGITS = 0); the CTA pair
    for 3- and 4-limb primes, the single CTA for 1-2 limbs (MHG_OPT_GEMM_KERNEL overrides); u8 chunks
    of (2^31 - 2^17) / (L * 255^2).  (Every combination's results are pinned by the
    parity tests.)"""
    opts(mh.OPT_DIGITS, 1)
    opts(mh.OPT_GEMM_KERNEL, 0)

    def variant(q, k, n=8192):
        lay, mod = mh.Layout(n, 64), mh.Modulus(q)
        A, B, C = (mh.Matrix(lay, mod) for _ in range(3))
        info = mh.Plan(mh.Problem(mh.Sub(A, 0, 256, 256), mh.Sub(B, 0, 256, k),
                                  mh.Sub(C, 0, k, 256)), mh.OP_SUB).info()
        return info["digits"], info["cta_group"], info["k_chunks"]

    assert variant(P16, 8192) == ("u8", 1, 1)
    assert variant(P16, 1024) == ("u8", 1, 1)
    assert variant(P31, 8192) == ("u8", 2, 1)
    assert variant(P24, 1024) == ("u8", 2, 1)
    assert variant(97, 512) == ("u8", 1, 1)
    assert variant(P16, 16384, n=16384) == ("u8", 1, 1)   # 16,384 = one u8 chunk at L = 2
    assert variant(P31, 16384, n=16384) == ("u8", 2, 2)   # 8,256 per chunk at L = 4
    opts(mh.OPT_DIGITS, 0)
    assert variant(P16, 8192)[0] == "s8"
    assert variant(P31, 16384, n=16384) == ("s8", 2, 1)
    opts(mh.OPT_GEMM_KERNEL, 1)
    assert variant(P31, 1024)[1] == 1


@pytest.mark.parametrize("q", [P16, P31, 97])
def test_device_verify(gpu, mh, oracle, q):
    """mhg_verify (Freivalds on the device): accepts every exact result -- ADD / SUB /
    SET, misaligned views -- and rejects a result with one corrupted view cell."""
    import torch
    rng = np.random.default_rng(q)
    n, t = 512, 32
    rounds = 2 if q > 1000 else 12
    for op in (OP_ADD, OP_SUB, OP_SET):
        r, k, c, corners = _random_views(rng, n)
        v = _views_from(oracle, n, t, r, k, c, corners)
        out, lhs, rhs = _fill(oracle, 500 + op, n, q)
        A, B, Cm, old = _containers(mh, n, t, q, (out, lhs, rhs, out))
        prob = mh.Problem(mh.Sub(A, v.out_origin, v.rows, v.cols), mh.Sub(B, v.lhs_origin, v.rows, v.inner),
                          mh.Sub(Cm, v.rhs_origin, v.inner, v.cols))
        mh.mm(prob, op)
        old_view = mh.Sub(old, v.out_origin, v.rows, v.cols)
        assert mh.verify(prob, old_view, op, rounds=rounds)
        # corrupt one cell inside the view
        cells = A.cells()
        z = oracle.encode(n, t, corners[0] + r // 2, corners[1] + c // 2)
        cells[z] = (int(cells[z]) + 1) % q
        A.upload(cells)
        assert not mh.verify(prob, old_view, op, rounds=rounds)
    torch.cuda.synchronize()


def test_device_verify_north_star(gpu, mh):
    """mhg_verify at the bench size (n = 16384, C -= A.B): exact result accepted."""
    import torch
    n, t, q = 16384, 64, P16
    g = torch.Generator(device="cuda").manual_seed(7)
    f = [torch.randint(0, q, (n * n,), dtype=torch.int32, device="cuda", generator=g) for _ in range(3)]
    f0 = f[0].clone()
    lay, mod = mh.Layout(n, t), mh.Modulus(q)
    A, B, Cm, old = (mh.Matrix.wrap(lay, mod, x.data_ptr(), owner=x) for x in (f[0], f[1], f[2], f0))
    prob = mh.Problem(mh.Sub(A, 0, n, n), mh.Sub(B, 0, n, n), mh.Sub(Cm, 0, n, n))
    mh.mm(prob, OP_SUB)
    assert mh.verify(prob, mh.Sub(old, 0, n, n), OP_SUB)
    f[0][12345] = (f[0][12345] + 1) % q
    assert not mh.verify(prob, mh.Sub(old, 0, n, n), OP_SUB)


def test_capture_refused_by_mm_accepted_for_plans(gpu, mh, oracle):
    """mhg_mm may grow its workspace (allocate + synchronise), so it refuses a capturing
    stream with MHG_ERR_UNSUPPORTED; a plan replayed inside a user's CUDA graph capture
    works and gives the exact result."""
    import torch
    n, t, q = 256, 32, P16
    out, lhs, rhs = _fill(oracle, 41, n, q)
    A, B, Cm = _containers(mh, n, t, q, (out, lhs, rhs))
    v = _views_from(oracle, n, t, 200, 150, 100, (3, 5, 7, 11, 13, 17))
    prob = mh.Problem(mh.Sub(A, v.out_origin, v.rows, v.cols), mh.Sub(B, v.lhs_origin, v.rows, v.inner),
                      mh.Sub(Cm, v.rhs_origin, v.inner, v.cols))
    plan = mh.Plan(prob, OP_SUB)
    plan.run()
    torch.cuda.synchronize()
    A.upload(out)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    refused = False
    with torch.cuda.graph(g, stream=s):
        try:
            mh.mm(prob, OP_SUB, stream=s)
        except mh.Unsupported:
            refused = True
        plan.run(s)
    assert refused
    g.replay()
    torch.cuda.synchronize()
    want = out.copy()
    oracle.mm_dense(n, t, q, want, lhs, rhs, v, op=OP_SUB)
    assert np.array_equal(A.cells(), want)


def test_upload_adaptive_raw_tail(gpu, mh, opts):
    """MHG_OPT_UPLOAD_ADAPTIVE: chunks of a pinned upload that travel raw (4-byte) while
    the link idles leave the container byte-identical to a plain copy, also with a wide
    cell (the rest then goes 4-byte) and for range uploads; PCIe bytes within [2, 4] per
    cell."""
    import torch
    opts(mh.OPT_UPLOAD_ADAPTIVE, 1)
    n, t, q = 8192, 64, P16
    rng = np.random.default_rng(91)
    m = mh.Matrix(mh.Layout(n, t), mh.Modulus(q))
    for bad in ([], [n * n // 3]):
        cells = rng.integers(0, q, size=n * n, dtype=np.uint32)
        for b in bad:
            cells[b] = 0x12345678
        h = torch.from_numpy(cells.view(np.int32)).pin_memory()
        s = torch.cuda.Stream()
        for _ in range(2):
            mh._check(mh.lib().mhg_matrix_upload(m.handle, h.data_ptr(), s.cuda_stream))
        s.synchronize()
        assert np.array_equal(m.cells(), cells)
        assert 2 * n * n <= m.upload_bytes <= 4 * n * n
    off, cnt = 12345, 20_000_000
    part = rng.integers(0, q, size=cnt, dtype=np.uint32)
    hp = torch.from_numpy(part.view(np.int32)).pin_memory()
    want = m.cells()
    mh._check(mh.lib().mhg_matrix_upload_range(m.handle, hp.data_ptr(), off, cnt, None))
    want[off:off + cnt] = part
    assert np.array_equal(m.cells(), want)


@pytest.mark.slow
@pytest.mark.parametrize("udig", [None, 0])
def test_general_fold_prime_at_chunk_limits(gpu, mh, opts, udig):
    """A 2-limb prime with 2^16 mod q >= 256 (q = 40961) takes the per-class fold and the
    fixed TMEM layout (no early release): extreme residues at one full exact chunk, one
    slice past it and a long K, ADD / SUB / SET, C_old = q - 1, closed form."""
    import torch
    if udig is not None:
        opts(mh.OPT_DIGITS, udig)
    q = 40961
    n, t, rows, cols = 32768, 64, 512, 512
    bufs = [torch.empty(n * n, dtype=torch.int32, device="cuda") for _ in range(3)]
    try:
        kc = _u8_chunk_slices(q) * 128
        for k in sorted({kc, kc + 128, 32768}):
            for x, y in [(0x9FFF, 0x9FFF), (0x9FFF, q - 1), ((q - 1) // 2, (q + 1) // 2)]:
                for op in (OP_ADD, OP_SUB, OP_SET):
                    a = (q - x) % q if op == OP_SUB else x
                    _device_constant_case(mh, n, t, q, a, y, q - 1, rows, k, cols, op, bufs)
    finally:
        del bufs
        torch.cuda.empty_cache()
