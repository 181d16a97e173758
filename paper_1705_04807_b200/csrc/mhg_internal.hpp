// mhg_internal.hpp -- types shared by the host planner (mhg_host.cpp) and the
// sm_100a kernels (mhg_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cstdint>

namespace mhg {

// ---------------------------------------------------------------- geometry
// Tile side of the Morton-hybrid layout (layout.hpp:42-76).  `shift` is
// log2(t) when t is a power of two, else -1 (non-pow2 tiles such as
// Layout(24, 3) are legal in the reference, layout_test.cpp:23).
struct TileGeom {
    uint64_t t;
    uint64_t tt;  // t * t
    int shift;
};

// ------------------------------------------------------------------ limbs
// Residues are mapped to a signed representative x' (x' == x mod q) and split
// into L signed 8-bit digits: x' = sum_s d_s 256^s, d_s in [-128, 127].
// Representative: x' = x if x <= H else x - q.  With H = min((q-1)/2,
// 127 (256^L - 1)/255) every x' fits L s8 digits whenever q <= 256^L.
struct DigitParams {
    uint32_t q;
    uint32_t H;
    int negate;  // 1: encode (q - x) mod q (C -= A.B as C += (-A).B)
    int udig;    // unsigned digits: x = sum_s d_s 256^s, d_s in [0, 255] (u8 x u8 MMA)
};

struct LimbParams {
    uint32_t L;          // digits per residue (1..4)
    uint32_t H;          // representative threshold
    uint32_t bound[4];   // max |digit| per position
    uint64_t k_max;      // max inner length with every int32 class sum <= 2^31 - 2^17
};

LimbParams limb_params(uint32_t q);

// ------------------------------------------------------------------- GEMM
// CTA tile: BM = 128 output rows x W output columns, W = 128 (L <= 2) or 64.
// K staged in BK-byte slices (one swizzle-atom row).  BK = 128 (SWIZZLE_128B):
// BK = 64 would allow a deeper ring of smaller stages, but SWIZZLE_64B operands
// slow the tensor pipe by ~20% (profiles/r01_ab_ring.txt).
constexpr int kBM = 128;
constexpr int kBK = 128;       // bytes of K per pipeline stage = one SWIZZLE_128B atom row
constexpr int kPackK = 128;    // K elements per k_pack_rows block
constexpr int kPackRows = 32;  // pack kernel block rows

inline int tile_width(int L) { return L <= 2 ? 128 : 64; }

struct GemmParams {
    const int8_t* apack;  // [Mt][Kt][L][128][128] swizzled
    const int8_t* bpack;  // [Nt][Kt][L][W][128]  swizzled
    uint32_t* out;        // Morton-hybrid container cells
    const uint64_t* out_rowoff;  // rows entries
    const uint64_t* out_coloff;  // cols entries
    uint64_t rows, cols;
    uint64_t out_i0, out_j0;     // view origin in the output container
    TileGeom out_geom;           // output container tile geometry (offsets in-kernel)
    uint32_t Mt, Nt, Kt, KC;     // KC: k-tiles per exact int32 chunk
    uint32_t q;
    uint32_t w32;                // 2^32 mod q
    uint64_t mu;                 // floor((2^64 - 1) / q)
    uint64_t bias;               // multiple of q >= 2^62 (signed -> unsigned shift)
    // 32-bit fold (L <= 2, q <= 2^16): class sums obey |a_c| <= 2^31 - 2^17
    uint32_t m32;                // floor(2^32 / q)
    uint32_t nq;                 // 2^32 - q (u - t q == u + t nq mod 2^32: one IMAD)
    uint32_t bias32;             // q * floor(2^31 / q): a_c + bias32 in [0, 2^32)
    uint32_t w16;                // 2^16 mod q
    int w16_small;               // w16 < 256: fold the top class without a mulmod
    int fold;                    // lean L = 2 fold level 3 / 2 / 1 (reductions per element; host)
    int mode;                    // 0: out += prod, 2: out = prod (first chunk)
    int udig;                    // unsigned (u8) digits: non-negative class sums (DigitParams::udig)
    int vec_ok;                  // t % 4 == 0: 16-byte epilogue accesses allowed
    uint32_t group;              // raster: row tiles per group sharing rhs panels in L2
    int keep_b;                  // rhs stages evict_last too (both packed operands fit in L2)
    int narrow;                  // 128 x 64 tiles (GemmGeometry::narrow)
    uint32_t wait_hint;          // mbarrier try_wait suspend-time hint, ns (k_gemm roles)
    unsigned long long* stats;   // optional per-CTA wait-cycle counters (diagnostics), or null
};

// k_gemm diagnostics layout (per CTA, when GemmParams::stats != null)
enum GemmStat { kStatTotal = 0, kStatMmaWaitFull, kStatMmaWaitTmem, kStatProdWaitEmpty,
                kStatEpiWaitFull, kStatEpiBusy, kStatEpiPrologue, kStatEpiTail, kStatEpiLdWait, kStatEpiIssue,
                kStatEpiLand, kStatCount };

// --------------------------------------------------------------- launchers
// All asynchronous on `stream`; return a cudaError_t value (0 = success).
int launch_offsets(uint64_t* dst, uint64_t start, uint64_t count, TileGeom g, int is_row,
                   void* stream);
// LDG/STG conversions; morton = 1 takes the Morton-order kernel where eligible.
int launch_rm_to_mh(const uint32_t* rm, uint32_t* mh, uint64_t n, TileGeom g, uint32_t q,
                    int* bad_flag, int morton, void* stream);
int launch_mh_to_rm(const uint32_t* mh, uint32_t* rm, uint64_t n, TileGeom g, int morton, void* stream);
// K1 through the TMA: `tmap` is a CUtensorMap over the row-major buffer (uint32, n x n,
// box t columns x R rows with R * t * 4 <= 16 KB; conv_tma_box_rows); power-of-two
// 4 <= t <= 256.  to_mh = 1 also checks residues < q (*bad).
int launch_conv_tma(const void* tmap, uint32_t* mh, uint64_t n, TileGeom g, uint32_t q, int* bad,
                    int to_mh, int num_sms, void* stream);
int conv_tma_smem();  // dynamic shared memory of the TMA conversion kernel
inline uint32_t conv_tma_box_rows(uint64_t t) {
    uint32_t R = (uint32_t)t;
    while ((uint64_t)R * t * 4 > 16384) R >>= 1;
    return R;
}
// Pack an operand into limb planes.  trans = 0: pack rows are view rows, K is
// view columns (lhs).  trans = 1: pack rows are view columns, K is view rows
// (rhs, transposed to K-major).  rows_per_tile = 128 (lhs) or W (rhs).
int launch_pack(int L, int trans, const uint32_t* src, const uint64_t* rowoff,
                const uint64_t* coloff, int vecok, uint64_t R, uint64_t K, uint32_t rows_per_tile,
                uint32_t Rtiles, uint32_t Kt, int8_t* dst, DigitParams dp, void* stream);
// One operand's pack job (launch_pack's arguments; Rpad is derived).
struct PackArgs {
    const uint32_t* src;
    const uint64_t* rowoff;
    const uint64_t* coloff;
    int vecok;
    uint64_t R, K;
    uint32_t rpt, Rtiles, Kt;
    uint64_t Rpad;
    int8_t* dst;
    DigitParams dp;
};
// lhs (rows, trans = 0) and rhs (cols, trans = 1) packs of one multiply in one launch.
int launch_pack_pair(int L, const PackArgs& lhs, const PackArgs& rhs, void* stream);
int launch_gemm(int L, const GemmParams& p, int num_sms, void* stream);
int gemm_smem_bytes(int L);
int diag_build();  // 1 when the kernels carry the wait-cycle counters (-DMHG_DIAG=1)
int configure_kernels();  // one-time kernel attributes (dynamic smem opt-in)
// CTA-pair GEMM: tmA / tmB point to CUtensorMap (2D uint8, rows of 128 B; box
// 128 rows for A, gemm2_b_box_rows(L) rows for B'); requires p.Mt even.
int launch_gemm2(int L, const GemmParams& p, const void* tmA, const void* tmB, int num_sms,
                 void* stream);
int gemm2_b_box_rows(int L);
int launch_widen16(const uint16_t* src, uint32_t* dst, uint64_t count, int num_sms,
                    void* stream);
// 16-bit upload wire (mhg_wire.cpp): true when uploads of this container size
// and modulus take it (q <= 2^16, >= 4M cells, not disabled by MHG_UPLOAD_WIRE=32).
bool wire16_enabled(uint32_t q, uint64_t count);
// Upload `count` host cells into cells[offset, offset + count): uint16 through pinned
// staging + k_widen16 while the cells fit 16 bits, plain 4-byte copies for the rest.
// *dev16 is the container's uint16 scratch of `total` cells (allocated here on first
// use; the caller frees it).  Returns a cudaError_t value; *wire_bytes = PCIe bytes.
int upload_wire16(uint32_t* cells, uint16_t** dev16, uint64_t total, uint64_t offset,
                  const uint32_t* host, uint64_t count, int num_sms, void* stream,
                  uint64_t* wire_bytes);
int launch_fill_view(uint32_t* out, const uint64_t* rowoff, const uint64_t* coloff, uint64_t rows,
                     uint64_t cols, uint32_t value, void* stream);
// Freivalds verification (mhg_verify): y = M x mod q over a view, a random vector, and
// the comparison of C_new r with C_old r +/- A (B r) (mode 0 add, 1 sub, 2 set).
int launch_matvec(const uint32_t* m, const uint64_t* rowoff, const uint64_t* coloff, uint64_t rows,
                  uint64_t cols, const uint32_t* x, uint32_t* y, uint32_t q, int num_sms, void* stream);
int launch_random_vec(uint32_t* r, uint64_t n, uint64_t seed, uint32_t q, void* stream);
int launch_freivalds_cmp(const uint32_t* wn, const uint32_t* wo, const uint32_t* z, uint64_t rows, uint32_t q,
                         int mode, int* bad, void* stream);

}  // namespace mhg

namespace mhg {

// ------------------------------------------------------------------ options
// Process-wide switches of the planner and test hooks (mhg_set_option, include/mhg.h).
// Initial values come from the environment, read once (mhg_options.cpp); after that
// only mhg_set_option changes them, so a stray variable cannot flip a kernel mid-run.
enum OptionKey {
    kOptDigits = 1,       // 1 = unsigned u8 limb digits, 0 = balanced s8
    kOptGemmKernel = 2,   // 0 = planner, 1 = single CTA, 2 = CTA pair
    kOptMinFold = 3,      // lowest lean-fold level the L = 2 epilogue may use (1..3)
    kOptMaxKChunk = 4,    // cap on K slices per exact chunk (0 = planner's bound)
    kOptUploadWire = 5,   // 0 = auto (by host workers), 16 = uint16 wire, 32 = 4-byte copies
    kOptConvKernel = 6,   // 0 = TMA where eligible, 1 = Morton-order LDG/STG, 2 = row-order
    kOptGemmStats = 7,    // 1 = per-launch wait-cycle report (synchronous diagnostics)
    kOptUploadThreads = 8,  // host narrowing workers (0 = affinity / LOCAL_WORLD_SIZE)
    kOptUploadAdaptive = 9, // 1 = idle-link chunks of a pinned upload travel raw (4-byte)
    kOptCount = 10
};
int64_t option(int key);
bool option_valid(int key, int64_t value);
void set_option(int key, int64_t value);

}  // namespace mhg
