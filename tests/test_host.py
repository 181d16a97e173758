"""Host-side tests (no GPU): the C-ABI library loads and exports every symbol
include/mhg.h declares, the planner's closed-form Counters equal the
reference's recursion, the limb representation is exact with the int32
bound the planner claims, and device entry points fail loudly (no CPU
fallback) when there is no B200."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "mhg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mhg_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(mh):
    lib = ctypes.CDLL(mh.LIB_PATH)
    syms = _declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_types_every_declared_entry_point(mh):
    """Every function include/mhg.h declares has explicit ctypes argument / result types in
    the Python mirror (an untyped call would pass 64-bit values as C ints)."""
    L = mh.lib()
    untyped = [n for n in _declared_symbols() if getattr(L, n).argtypes is None]
    assert not untyped, untyped


def test_header_is_plain_c(tmp_path):
    """include/mhg.h is a C header (the drop-in boundary is a C ABI): it compiles as strict
    C11 on its own, every struct and handle type usable from C."""
    import subprocess
    src = tmp_path / "abi.c"
    src.write_text('#include "mhg.h"\n'
                   "int main(void) { mhg_view v = {0, 0, 0, 0}; mhg_counters c; mhg_dist_block_t b;\n"
                   "  mhg_dist_segment_t s; mhg_ipc_handle h; mhg_plan p = 0; mhg_sweep w = 0; mhg_matrix m = 0;\n"
                   "  (void)v; (void)c; (void)b; (void)s; (void)h; (void)p; (void)w; (void)m;\n"
                   "  return (int)MHG_OK; }\n")
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I",
                        os.path.join(ROOT, "include"), "-fsyntax-only", str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_no_torch_types_in_abi():
    src = open(os.path.join(ROOT, "include", "mhg.h")).read()
    assert "torch" not in src.split("*/", 1)[1]
    assert "cudaStream_t" not in re.sub(r"/\*.*?\*/", "", src, flags=re.S)


def test_layout_and_modulus_validation(mh):
    """layout_test.cpp:20-28, field_test.cpp:10-19, layout_test.cpp:100-106."""
    mh.Layout(8, 4), mh.Layout(1, 1), mh.Layout(24, 3)
    for n, t in [(8, 3), (12, 4), (0, 1), (8, 0)]:
        with pytest.raises(mh.InvalidArgument):
            mh.Layout(n, t)
    for q in (0, 1, 9, 2 ** 31, 65535):
        with pytest.raises(mh.InvalidArgument):
            mh.Modulus(q)
    mh.Modulus(2), mh.Modulus(65521), mh.Modulus(2147483647)
    lay = mh.Layout(8, 4)
    assert mh.encode(lay, 2, 5) == 25 and mh.encode(lay, 5, 6) == 54
    assert (mh.extract_i(lay, 47), mh.extract_j(lay, 47)) == (7, 3)
    with pytest.raises(mh.OutOfRange):
        mh.encode(lay, 8, 0)
    with pytest.raises(mh.OutOfRange):
        mh.extract_i(lay, 64)


def test_codec_matches_oracle(mh, oracle):
    for n, t in [(16, 4), (24, 3), (256, 32), (4096, 64)]:
        lay = mh.Layout(n, t)
        rng = np.random.default_rng(n)
        for _ in range(200):
            i, j = (int(x) for x in rng.integers(0, n, 2))
            z = mh.encode(lay, i, j)
            assert z == oracle.encode(n, t, i, j)
            assert (mh.extract_i(lay, z), mh.extract_j(lay, z)) == (i, j)


def test_planner_counters_equal_reference(mh, oracle, reference):
    """Closed-form Counters (all five fields) == the reference's recursion."""
    rng = np.random.default_rng(3)
    for it in range(400):
        n = int(rng.choice([8, 16, 32, 64, 128]))
        t = int(rng.choice([x for x in (1, 2, 4, 8, 16, 32) if x <= n]))
        if it % 9 == 0:
            n, t = 48, 3
        q = 2
        out, lhs, rhs, _, v = oracle.gen_problem(oracle.rng(it), n, t, q)
        got = mh.counters_layout(n, t, v.out_origin, v.lhs_origin, v.rhs_origin, v.rows, v.inner,
                                 v.cols)
        want = reference.mm_oblivious(n, t, q, out.copy(), lhs, rhs, v)
        assert got.as_tuple() == want.as_tuple(), (n, t, v)


def test_planner_counters_golden(mh):
    """Reference-generated golden cases (tests/golden/cases.json) and the
    20-trial batch of bench_test.cpp (oblivious calls + macs columns)."""
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "cases.json")))
    for c in gold:
        o, l, r, rows, inner, cols = c["views"]
        got = mh.counters_layout(c["n"], c["t"], o, l, r, rows, inner, cols)
        assert list(got.as_tuple()) == c["counters"]
    csv = open(os.path.join(ROOT, "tests", "golden", "bench_trials_seed0_n64_t8_q2.csv")).read()
    for ln in csv.strip().splitlines()[1:]:
        f = [int(x) for x in ln.split(",")]
        got = mh.counters_layout(64, 8, f[1], f[4], f[7], f[2], f[6], f[3])
        assert (got.base_case_calls, got.scalar_macs) == (f[11], f[12])


def test_baseline_config_leaf_counts(mh):
    """SURVEY 8(a) leaf counts at the BASELINE configurations."""
    c = mh.counters_layout(512, 32, 0, 0, 0, 512, 512, 512)
    assert c.base_case_calls == 16 ** 3 and c.recursive_calls == 1 + 8 + 64 + 512 + 4096
    lay = mh.Layout(8192, 64)
    z = mh.encode(lay, 96, 160)
    c = mh.counters_layout(8192, 64, z, z, z, 6144, 2048, 5120)
    assert c.base_case_calls == 97 * 33 * 81
    c = mh.counters_layout(32768, 64, 0, 0, 0, 32768, 32768, 32768)
    assert c.base_case_calls == 512 ** 3 and c.scalar_macs == 32768 ** 3


def _digits(v, q, H, L, negate=False):
    """Python restatement of the device digit split (mhg_kernels.cu to_digits)."""
    if negate:
        v = (q - v) % q
    x = v if v <= H else v - q
    d = []
    for _ in range(L - 1):
        lo = ((x & 0xFF) ^ 0x80) - 0x80
        d.append(lo)
        x = (x - lo) >> 8
    d.append(x)
    return d


@pytest.mark.parametrize("q", [2, 3, 97, 251, 257, 65521, 65537, 16777213, 16777259,
                               2147483629, 2147483647])
def test_limb_representation_exact(mh, q):
    L, H, kmax = mh.limb_params(q)
    assert q <= 256 ** L and (L == 1 or q > 256 ** (L - 1))
    rng = np.random.default_rng(q % 1000)
    vals = {0, 1, q - 1, q // 2, q // 2 + 1, H, min(H + 1, q - 1)} | set(
        int(x) for x in rng.integers(0, q, 3000))
    vals = {v for v in vals if v < q}
    top = 0
    for v in vals:
        for neg in (False, True):
            d = _digits(v, q, H, L, neg)
            assert all(-128 <= x <= 127 for x in d), (v, d)
            val = sum(x * 256 ** s for s, x in enumerate(d))
            assert val % q == ((q - v) % q if neg else v)
            top = max(top, abs(d[-1]))
    # the planner's K bound keeps every int32 class sum exact
    bound = [128] * (L - 1) + [top]
    worst = max(sum(bound[s] * bound[c - s] for s in range(L) if 0 <= c - s < L)
                for c in range(2 * L - 1))
    assert kmax * worst <= 2 ** 31 - 1


def test_north_star_fits_one_chunk(mh):
    """p=65521 needs 2 limbs and keeps K=32768 (cfg5) in one exact chunk;
    p=2^31-1 needs 4 limbs and fits K=8192 (cfg4)."""
    L, H, kmax = mh.limb_params(65521)
    assert L == 2 and kmax >= 32768
    L, H, kmax = mh.limb_params(2147483647)
    assert L == 4 and kmax >= 8192


def test_device_calls_fail_loudly_without_gpu(mh):
    """No CPU fallback: without an sm_100 device every compute entry point raises."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(mh.DeviceError):
        mh.Matrix(mh.Layout(8, 4), mh.Modulus(2))
    assert mh.lib().mhg_device_check() != 0


# ---- fold levels of the 2-limb epilogue (mhg_fold_level; kernel fold_g1 / fold_g2)
M32 = 0xFFFFFFFF


def _emulate_fold(level, layout, a0, a1, a2, cur, q, bias32=None):
    """Bit-exact emulation of the kernel's lean L=2 fold (uint32 wrap-around,
    Barrett red32 with m = floor(2^32 / q), csrc/mhg_kernels.cu fold_g1/fold_g2).
    bias32 = GemmParams::bias32 (0 for unsigned-digit plans)."""
    w16 = (1 << 16) % q
    m32 = (1 << 32) // q
    if bias32 is None:
        bias32 = ((1 << 31) // q) * q

    def red32(u):
        u &= M32
        r = (u - ((u * m32) >> 32) * q) & M32
        return r - q if r >= q else r

    def sra8(v):  # arithmetic shift of an int32
        return v >> 8

    x, y, z = (a1, a2, a0) if layout == 0 else (a0, a1, a2)
    if level <= 2:
        if layout == 0:
            lo = (x & 0xFF) << 8
            if level == 1:
                g1 = lo + w16 * ((sra8(x) + y) & M32)
            else:
                g1 = lo + w16 * (((sra8(x) & M32) + red32(y + bias32)) & M32)
        else:
            g1 = x + ((y & 0xFF) << 8) + w16 * (sra8(y) & M32)
    else:
        r1 = red32((y if layout else x) + bias32)
        g1 = ((r1 << 8) + w16 * red32(y + bias32)) if layout == 0 else (x + bias32 + (r1 << 8))
    c = (cur + g1) & M32
    if layout == 0:
        return red32(c + z + bias32)
    if level == 1:
        return red32(c + w16 * (z & M32) + bias32)
    r2 = red32(z + bias32)
    return red32(c + w16 * r2 + bias32) if level == 2 else red32(c + w16 * r2)


@pytest.mark.parametrize("q", [65521, 65519, 65287, 257, 3])
def test_fold_levels_exact_at_their_bounds(mh, q):
    """For each fold level the host admits, the kernel arithmetic (emulated bit
    for bit) is exact at the largest admitted chunk with extreme class sums."""
    L, H, kmax = mh.limb_params(q)
    if L != 2:
        assert mh.fold_level(q, 128) == 3
        return
    rng = np.random.default_rng(q)
    # largest |top digit| of any representative (the low digit spans [-128, 127])
    top = max(abs(_digits(v, q, H, L, neg)[-1]) for v in range(q) for neg in (False, True)) \
        if q < 70000 else 128
    for level in (1, 2, 3):
        lo, hi = 0, kmax  # largest K with fold_level(q, K) <= level
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if mh.fold_level(q, mid) <= level:
                lo = mid
            else:
                hi = mid - 1
        K = lo
        if K == 0:
            continue
        # class-sum magnitudes reachable with chunk K (products of digits)
        e0, e1, e2 = 128 * 128 * K, 2 * 128 * top * K, top * top * K
        cases = [(s0 * e0, s1 * e1, s2 * e2) for s0 in (-1, 1) for s1 in (-1, 1) for s2 in (-1, 1)]
        cases += [(int(rng.integers(-e0, e0 + 1)), int(rng.integers(-e1, e1 + 1)),
                   int(rng.integers(-e2, e2 + 1))) for _ in range(300)]
        for a0, a1, a2 in cases:
            for cur in (0, q - 1, int(rng.integers(0, q))):
                want = (cur + a0 + 256 * a1 + 65536 * a2) % q
                for layout in (0, 1):
                    got = _emulate_fold(level, layout, a0, a1, a2, cur, q)
                    assert got == want, (q, level, K, layout, a0, a1, a2, cur)


def test_fold_level_choices(mh):
    """p = 65521: one reduction up to K = 8064 (63 k-tiles), two beyond; a prime
    with 2^16 mod q >= 256 always takes the per-class fold."""
    assert mh.fold_level(65521, 1024) == 1
    assert mh.fold_level(65521, 8064) == 1
    assert mh.fold_level(65521, 8192) == 2
    assert mh.fold_level(65521, 65408) == 2
    assert mh.fold_level(65287, 512) == 1 and mh.fold_level(65287, 640) == 2
    q = 40009  # 2^16 mod q = 25527
    assert (1 << 16) % q >= 256 and mh.fold_level(q, 128) == 3
    assert mh.fold_level(2147483647, 128) == 3


@pytest.mark.parametrize("q", [65521, 65519, 65287, 257, 40009])
def test_fold_levels_u8_exact_at_their_bounds(mh, q):
    """Unsigned (u8) digits: class sums in [0, 255^2 k] / [0, 2 * 255^2 k] / [0, 255^2 k],
    no bias.  For each level mhg_fold_level_u8 admits, the emulated kernel arithmetic is
    exact at the largest admitted chunk (up to the u8 chunk bound (2^31 - 2^17) / (2 * 255^2))."""
    kmax_u = ((1 << 31) - (1 << 17)) // (2 * 65025)
    rng = np.random.default_rng(q + 1)
    seen = set()
    for level in (1, 2, 3):
        lo, hi = 0, kmax_u
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if mh.fold_level(q, mid, unsigned_digits=True) <= level:
                lo = mid
            else:
                hi = mid - 1
        K = lo
        if K == 0:
            continue
        seen.add(level)
        e0, e1, e2 = 65025 * K, 2 * 65025 * K, 65025 * K
        cases = [(b0 * e0, b1 * e1, b2 * e2) for b0 in (0, 1) for b1 in (0, 1) for b2 in (0, 1)]
        cases += [(int(rng.integers(0, e0 + 1)), int(rng.integers(0, e1 + 1)),
                   int(rng.integers(0, e2 + 1))) for _ in range(300)]
        for a0, a1, a2 in cases:
            for cur in (0, q - 1, int(rng.integers(0, q))):
                want = (cur + a0 + 256 * a1 + 65536 * a2) % q
                for layout in (0, 1):
                    got = _emulate_fold(level, layout, a0, a1, a2, cur, q, bias32=0)
                    assert got == want, (q, level, K, layout, a0, a1, a2, cur)
    if (1 << 16) % q < 256:
        assert 2 in seen  # every u8 chunk has a lean fold
    else:
        assert seen == {3}


def test_naive_default_counters_equal_reference(mh, reference):
    """mm_naive / mm_default Counters (multiply.hpp:269-291) in closed form -- incl.
    max_consecutive_jump of their encode-addressed walks (:80-129) -- equal the
    reference's own on random problems whose three containers differ in n and t (the
    two kernels have no layout guard), power-of-two and other tile sides."""
    rng = np.random.default_rng(20261020)
    for _ in range(300):
        geos = []
        for _ in range(3):
            t = int(rng.choice([1, 2, 3, 4, 5, 8, 16]))
            geos.append((t << int(rng.integers(0, 4)), t))
        r = int(rng.integers(1, min(geos[0][0], geos[1][0]) + 1))
        c = int(rng.integers(1, min(geos[0][0], geos[2][0]) + 1))
        k = int(rng.integers(1, min(geos[1][0], geos[2][0]) + 1))

        def corner(g, rows, cols):
            n, t = g
            return (n, t, mh.encode(mh.Layout(n, t), int(rng.integers(0, n - rows + 1)),
                                    int(rng.integers(0, n - cols + 1))))
        go, gl, gr = corner(geos[0], r, c), corner(geos[1], r, k), corner(geos[2], k, c)
        for kind, flag in ((0, mh.KERNEL_NAIVE), (1, mh.KERNEL_DEFAULT)):
            want = reference.counters_mixed(kind, go, gl, gr, r, k, c).as_tuple()
            got = mh.counters_geometry(flag, go, gl, gr, r, k, c).as_tuple()
            assert got == want, (kind, go, gl, gr, r, k, c)


def test_naive_default_counters_on_acceptance_draws(mh, oracle, reference):
    """The same on the reference's acceptance draws (gen_problem, same layouts), and the
    scattered default run of multiply_test.cpp:409-424 (jump > t, encodes > 0)."""
    for (n, t, seed, count) in [(64, 8, 11, 30), (128, 16, 12, 10), (96, 3, 13, 20)]:
        g = oracle.rng(seed)
        for _ in range(count):
            _, _, _, _, v = oracle.gen_problem(g, n, t, 2)
            for kind, flag in ((0, mh.KERNEL_NAIVE), (1, mh.KERNEL_DEFAULT)):
                want = reference.counters_mixed(kind, (n, t, v.out_origin), (n, t, v.lhs_origin),
                                                (n, t, v.rhs_origin), v.rows, v.inner, v.cols)
                got = mh.counters_geometry(flag, (n, t, v.out_origin), (n, t, v.lhs_origin),
                                           (n, t, v.rhs_origin), v.rows, v.inner, v.cols)
                assert got.as_tuple() == want.as_tuple()
    n, t = 64, 8
    s = mh.encode(mh.Layout(n, t), t // 2, t // 2)
    c = mh.counters_geometry(mh.KERNEL_DEFAULT, (n, t, s), (n, t, s), (n, t, s), 2 * t, 2 * t, 2 * t)
    assert c.max_consecutive_jump > t and c.encode_calls > 0


def test_product_rng_reproduces_reference_draws(mh, oracle):
    """mhg_rng (mh::Rng, bench.hpp:44-52) in the product library: the seed-0 first
    gen_problem draw of bench_test.cpp:56-72 (descriptor triple and the container hash
    4715125990397575263), and the same stream as the oracle's restatement."""
    g = mh.Rng(0)
    n = 64
    assert int(g.below(8)[0]) != 0  # uniform mode
    r, k, c = (1 + int(x) for x in g.below(n, 3))
    ia = int(g.below(n - r + 1)[0]); ja = int(g.below(n - c + 1)[0])
    ib = int(g.below(n - r + 1)[0]); jb = int(g.below(n - k + 1)[0])
    ic = int(g.below(n - k + 1)[0]); jc = int(g.below(n - c + 1)[0])
    lay = mh.Layout(n, 8)
    assert (mh.encode(lay, ia, ja), r, c) == (1, 64, 39)
    assert (mh.encode(lay, ib, jb), k) == (322, 3)
    assert mh.encode(lay, ic, jc) == 2855
    out = g.below(2, n * n)
    h = 0
    for x in out.tolist():
        h = (h * 31 + x) & (2 ** 64 - 1)
    assert h == 4715125990397575263
    a, b = mh.Rng(12345), oracle.rng(12345)
    assert np.array_equal(a.below(65521, 10000), oracle.fill_below(b, 10000, 65521))


def test_options_api(mh):
    """mhg_set_option / mhg_get_option: typed keys, range checks, restore; the GEMM
    wait counters exist only in diagnostic builds (MHG_ERR_UNSUPPORTED here)."""
    saved = {k: mh.get_option(k) for k in range(1, 10)}
    try:
        assert saved[mh.OPT_DIGITS] in (0, 1)
        mh.set_option(mh.OPT_DIGITS, 0)
        assert mh.get_option(mh.OPT_DIGITS) == 0
        mh.set_option(mh.OPT_MAX_KCHUNK, 3)
        assert mh.get_option(mh.OPT_MAX_KCHUNK) == 3
        for key, bad in [(mh.OPT_DIGITS, 2), (mh.OPT_GEMM_KERNEL, 3), (mh.OPT_MIN_FOLD_LEVEL, 0),
                         (mh.OPT_MIN_FOLD_LEVEL, 4), (mh.OPT_UPLOAD_WIRE, 8), (mh.OPT_CONV_KERNEL, 3),
                         (mh.OPT_MAX_KCHUNK, -1), (0, 0), (99, 0)]:
            with pytest.raises(mh.InvalidArgument):
                mh.set_option(key, bad)
        with pytest.raises(mh.InvalidArgument):
            mh.get_option(99)
        with pytest.raises(mh.Unsupported):  # product build: no wait-cycle counters
            mh.set_option(mh.OPT_GEMM_STATS, 1)
        with mh.options({mh.OPT_GEMM_KERNEL: 2, mh.OPT_DIGITS: 1}):
            assert mh.get_option(mh.OPT_GEMM_KERNEL) == 2
        assert mh.get_option(mh.OPT_GEMM_KERNEL) == saved[mh.OPT_GEMM_KERNEL]
    finally:
        for k, v in saved.items():
            mh.set_option(k, v)


def test_options_select_the_planner_choice(mh):
    """The options reach the planner: digits and K-chunk cap change the exact chunking
    reported by the host-only planner entry points (mhg_fold_level / counters are
    unaffected: results and Counters never depend on the options)."""
    c0 = mh.counters_layout(1024, 64, 0, 0, 0, 1024, 1024, 1024).as_tuple()
    with mh.options({mh.OPT_DIGITS: 0, mh.OPT_MAX_KCHUNK: 1}):
        assert mh.counters_layout(1024, 64, 0, 0, 0, 1024, 1024, 1024).as_tuple() == c0
