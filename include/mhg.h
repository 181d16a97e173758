/*
 * mhg.h -- C ABI of the B200-native Morton-hybrid GF(p) matrix-multiply path.
 *
 * This is the drop-in boundary.  The reference (arxiv/paper_1705_04807,
 * proj/include/mh) has no FFI: its interface is the header API
 * `mh::mm_oblivious(const Problem&) -> Counters` (multiply.hpp:297-308) over
 * three `Sub` views (submatrix.hpp:13-18) of `Matrix` containers
 * (matrix.hpp:13-39).  Each entry point below names the reference interface it
 * replaces.  A C++ mirror of the reference header API (namespace mh, same
 * names) is layered on top in include/mh/ (C++ headers); INTEGRATION.md shows the
 * bindings.
 *
 * Conventions
 *  - Plain C types only: no torch, no CUDA types.  `stream` is a cudaStream_t
 *    passed as void* (NULL = legacy default stream).
 *  - Every call returns an mhg_status; MHG_OK == 0.  The status codes map one
 *    to one onto the exception classes the reference throws
 *    (std::invalid_argument, std::out_of_range, std::logic_error); the message
 *    of the last failure on the calling thread is mhg_last_error().
 *  - Device work is asynchronous on `stream` unless the name says otherwise.
 *  - There is no CPU fallback: on a machine without an sm_100 GPU every compute
 *    entry point fails with MHG_ERR_DEVICE.
 */
#ifndef MHG_H
#define MHG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MHG_OK = 0,
    MHG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    MHG_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range */
    MHG_ERR_LOGIC = 3,            /* std::logic_error */
    MHG_ERR_DEVICE = 4,           /* CUDA failure / no sm_100 device */
    MHG_ERR_UNSUPPORTED = 5       /* valid for the reference, not for this build */
} mhg_status;

/* Operation applied to the output view.  The reference only accumulates
 * (multiply.hpp:9-10); SUB is the TU/TURBO Schur update C -= A*B and SET is
 * C = A*B (view cells only). */
typedef enum { MHG_OP_ADD = 0, MHG_OP_SUB = 1, MHG_OP_SET = 2 } mhg_op;

/* Opaque device-resident Morton-hybrid container (replaces mh::Matrix,
 * matrix.hpp:13-39): n x n uint32 residues mod q in the reference's flat
 * order (tile Z-index * t*t + row-major offset inside the tile,
 * layout.hpp:80-85), so uploads, downloads and parity compares are memcpys. */
typedef struct mhg_matrix_s *mhg_matrix;

/* Opaque reusable multiply plan (see mhg_plan_create). */
typedef struct mhg_plan_s *mhg_plan;

/* A view: the reference's Sub 4-tuple (M, sigma, r, c), submatrix.hpp:13-18. */
typedef struct {
    mhg_matrix mat;
    uint64_t origin; /* flat index of the first entry */
    uint64_t rows;
    uint64_t cols;
} mhg_view;

/* The reference's Counters (multiply.hpp:39-45), computed in closed form by
 * the planner for the oblivious decomposition (identical values). */
typedef struct {
    uint64_t base_case_calls;
    uint64_t scalar_macs;
    uint64_t encode_calls;
    uint64_t recursive_calls;
    uint64_t max_consecutive_jump;
} mhg_counters;

/* ---- errors / device ---- */
const char *mhg_last_error(void);
/* Fails with MHG_ERR_DEVICE unless the current device is sm_100. */
mhg_status mhg_device_check(void);
const char *mhg_version(void);

/* ---- options (process-wide; no reference counterpart) ----
 * The planner's kernel and digit choices and the test hooks.  Every value gives
 * bit-identical results; only speed differs.  Initial values are read ONCE, at the
 * first use, from the environment variable named beside each key; afterwards only
 * mhg_set_option changes them.  Unknown keys / out-of-range values fail with
 * MHG_ERR_INVALID_ARGUMENT. */
typedef enum {
    MHG_OPT_DIGITS = 1,          /* MHG_UDIG: 1 = unsigned u8 limb digits (default), 0 = balanced s8 */
    MHG_OPT_GEMM_KERNEL = 2,     /* MHG_GEMM: 0 = planner (single CTA for <= 2 limbs, CTA pair for
                                    3-4), 1 = single-CTA k_gemm, 2 = CTA-pair k_gemm2 */
    MHG_OPT_MIN_FOLD_LEVEL = 3,  /* MHG_FOLD: lowest lean-fold level of the 2-limb epilogue, 1..3 */
    MHG_OPT_MAX_KCHUNK = 4,      /* MHG_FORCE_KCHUNK: cap on 128-byte K slices per exact int32
                                    chunk (0 = the planner's bound; small values force multi-chunk K) */
    MHG_OPT_UPLOAD_WIRE = 5,     /* MHG_UPLOAD_WIRE: 0 = auto (16-bit wire with >= 8 host workers),
                                    16 = 16-bit wire where eligible, 32 = plain 4-byte copies */
    MHG_OPT_CONV_KERNEL = 6,     /* MHG_CONV: 0 = TMA where eligible (default), 1 = Morton-order
                                    LDG/STG, 2 = row-order LDG/STG */
    MHG_OPT_GEMM_STATS = 7,      /* MHG_GEMM_STATS: 1 = print per-launch wait-cycle shares to stderr
                                    (synchronous; diagnostics) */
    MHG_OPT_UPLOAD_THREADS = 8,  /* MHG_UPLOAD_THREADS: host narrowing workers (0 = the affinity
                                    mask / LOCAL_WORLD_SIZE) */
    MHG_OPT_UPLOAD_ADAPTIVE = 9  /* MHG_UPLOAD_ADAPTIVE: 1 = while the link idles (the host narrows
                                    slower than PCIe), chunks from the back of a PINNED source
                                    travel as 4-byte cells on a second copy stream */
} mhg_option;
mhg_status mhg_set_option(int key, int64_t value);
mhg_status mhg_get_option(int key, int64_t *value);

/* ---- layout codec (layout.hpp:42-99): host-side, no device needed ---- */
mhg_status mhg_layout_check(uint64_t n, uint64_t t);                 /* Layout(n,t) ctor :50-62 */
mhg_status mhg_encode(uint64_t n, uint64_t t, uint64_t i, uint64_t j, uint64_t *z); /* :80-85 */
mhg_status mhg_extract(uint64_t n, uint64_t t, uint64_t z, uint64_t *i, uint64_t *j); /* :88-99 */
mhg_status mhg_modulus_check(uint32_t q);                            /* Modulus(q), field.hpp:28-34 */

/* ---- containers (matrix.hpp) ---- */
/* Matrix(Layout(n,t), Modulus(q)): device allocation, zero filled. */
mhg_status mhg_matrix_create(uint64_t n, uint64_t t, uint32_t q, mhg_matrix *out);
/* Non-owning container over an existing device buffer of n*n uint32. */
mhg_status mhg_matrix_wrap(uint64_t n, uint64_t t, uint32_t q, void *device_cells, mhg_matrix *out);
mhg_status mhg_matrix_destroy(mhg_matrix m);
mhg_status mhg_matrix_info(mhg_matrix m, uint64_t *n, uint64_t *t, uint32_t *q, void **device_cells);
/* Flat Morton-hybrid order copies (Matrix::cells(), matrix.hpp:27-28). */
/* Upload: asynchronous on `stream` (the host buffer must stay valid until the
 * stream reaches the copy).  For q <= 2^16 and >= 4M cells the cells travel as
 * uint16 (half the PCIe bytes): host threads narrow them into pinned staging
 * while earlier chunks are in flight, and the device widens them; the call then
 * returns once the host buffer has been read.  Any cell >= 2^16 switches the
 * rest of the upload to 4-byte copies, so the container always equals a plain
 * copy of the buffer.  MHG_UPLOAD_WIRE=32 disables the 16-bit wire. */
mhg_status mhg_matrix_upload(mhg_matrix m, const uint32_t *host_cells, void *stream);
/* Upload of the flat cell range [offset, offset + count) from `host_cells` (which
 * holds exactly those cells), same wire rules; e.g. one rank's Morton slice. */
mhg_status mhg_matrix_upload_range(mhg_matrix m, const uint32_t *host_cells, uint64_t offset,
                                   uint64_t count, void *stream);
/* PCIe bytes moved by the last mhg_matrix_upload / _upload_range of `m`. */
mhg_status mhg_matrix_upload_bytes(mhg_matrix m, uint64_t *bytes);
mhg_status mhg_matrix_download(mhg_matrix m, uint32_t *host_cells, void *stream);
/* from_row_major / to_row_major (matrix.hpp:44-67) on DEVICE buffers of n*n
 * row-major uint32 (K1 conversion kernels).  from_row_major's residue check
 * (:52-53) is applied on the device: an out-of-range residue fails the call
 * with MHG_ERR_INVALID_ARGUMENT (synchronous on `stream`). */
mhg_status mhg_rowmajor_to_mh(mhg_matrix dst, const uint32_t *device_rows, void *stream);
mhg_status mhg_mh_to_rowmajor(mhg_matrix src, uint32_t *device_rows, void *stream);
/* Same two conversions from / to HOST row-major buffers (staged through a
 * device scratch buffer, K1 on the device); synchronous. */
mhg_status mhg_rowmajor_host_to_mh(mhg_matrix dst, const uint32_t *host_rows);
mhg_status mhg_mh_to_rowmajor_host(mhg_matrix src, uint32_t *host_rows);
/* cudaStreamSynchronize(stream) for callers that do not link the CUDA runtime. */
mhg_status mhg_synchronize(void *stream);
/* Streams for such callers: a cudaStream_t as void* on the current device (non_blocking != 0:
 * cudaStreamNonBlocking, i.e. not ordered with the default stream).  The reference allows
 * concurrent multiplies on disjoint output rectangles (multiply.hpp:25-29); here they run
 * on different streams. */
mhg_status mhg_stream_create(void **stream, int non_blocking);
mhg_status mhg_stream_destroy(void *stream);
/* Events (cudaEvent_t as void*, timing disabled) for the same callers: the C++ mirror's
 * Matrix orders asynchronous multiplies on different streams with them.  An event stays
 * valid after the stream it was recorded on is destroyed.  mhg_event_query: *done = 1 when
 * the work captured by the last record has completed. */
mhg_status mhg_event_create(void **event);
mhg_status mhg_event_record(void *event, void *stream);
mhg_status mhg_event_query(void *event, int *done);
mhg_status mhg_event_synchronize(void *event);
mhg_status mhg_stream_wait_event(void *stream, void *event);
mhg_status mhg_event_destroy(void *event);

/* ---- multiply (multiply.hpp) ---- */
/* out op= lhs * rhs over the three views, computed on the GPU with the int8
 * limb-split tcgen05 kernels.  Validation follows check_problem
 * (multiply.hpp:55-66) and mm_oblivious's layout guard (:299-301); an empty
 * problem is a no-op with zero Counters (:303).  `ctr` may be NULL.
 * Replaces mh::mm_oblivious (multiply.hpp:297-308). */
mhg_status mhg_mm(mhg_view out, mhg_view lhs, mhg_view rhs, mhg_op op, mhg_counters *ctr,
                  void *stream);

/* Extended form.  flags & MHG_ALLOW_ALIAS lifts the reference's distinct-
 * container rule (multiply.hpp:59-60) for the TU/TURBO Schur update, where
 * C, A and B are views of ONE parent: the operands are read (packed) before the
 * output is written, so the result is C_new = C_old op A_old * B_old even when
 * the views overlap.  All other checks are unchanged.
 * MHG_KERNEL_NAIVE / MHG_KERNEL_DEFAULT: the same GPU computation behind the
 * reference's other two entry points, mm_naive (multiply.hpp:269-278) and mm_default
 * (:283-291): their validation (no layout guard -- the three containers may differ in
 * n and t) and their Counters (closed form, incl. max_consecutive_jump). */
#define MHG_ALLOW_ALIAS 1u
#define MHG_KERNEL_NAIVE 2u
#define MHG_KERNEL_DEFAULT 4u
mhg_status mhg_mm_ex(mhg_view out, mhg_view lhs, mhg_view rhs, mhg_op op, uint32_t flags,
                     mhg_counters *ctr, void *stream);
mhg_status mhg_plan_create_ex(mhg_view out, mhg_view lhs, mhg_view rhs, mhg_op op, uint32_t flags,
                              mhg_plan *plan);

/* Counters only (no device work): the closed form of the oblivious recursion. */
mhg_status mhg_counters_oblivious(mhg_view out, mhg_view lhs, mhg_view rhs, mhg_counters *ctr);
/* Same, from the raw layout and view origins (three same-layout containers);
 * pure host planner, usable without a GPU. */
mhg_status mhg_counters_layout(uint64_t n, uint64_t t, uint64_t out_origin, uint64_t lhs_origin,
                               uint64_t rhs_origin, uint64_t rows, uint64_t inner, uint64_t cols,
                               mhg_counters *ctr);
/* Counters of the reference kernel selected by flags (0: mm_oblivious, MHG_KERNEL_NAIVE,
 * MHG_KERNEL_DEFAULT), with that kernel's validation; no device work. */
mhg_status mhg_counters_for(uint32_t flags, mhg_view out, mhg_view lhs, mhg_view rhs, mhg_counters *ctr);
/* The same from raw geometry: each container's (n, t) and the view's flat origin;
 * pure host code, usable without a GPU. */
mhg_status mhg_counters_geometry(uint32_t flags, uint64_t n_out, uint64_t t_out, uint64_t out_origin,
                                 uint64_t n_lhs, uint64_t t_lhs, uint64_t lhs_origin, uint64_t n_rhs,
                                 uint64_t t_rhs, uint64_t rhs_origin, uint64_t rows, uint64_t inner,
                                 uint64_t cols, mhg_counters *ctr);

/* Reusable plan: validation, offset tables, packing workspace and a captured
 * CUDA graph (pack lhs, pack rhs, GEMM + fused epilogue) replayed by
 * mhg_plan_run.  The views' containers must outlive the plan.  mhg_plan_run on a
 * stream that the caller is capturing enqueues the kernels themselves (they become
 * nodes of the caller's graph); mhg_mm refuses capture (MHG_ERR_UNSUPPORTED). */
mhg_status mhg_plan_create(mhg_view out, mhg_view lhs, mhg_view rhs, mhg_op op, mhg_plan *plan);
mhg_status mhg_plan_run(mhg_plan plan, void *stream);
/* Split execution of a plan, for exchanging PACKED operands between ranks
 * (multi-GPU: 2-byte limb planes instead of uint32 cells):
 *   mhg_plan_pack        pack one operand of the plan's views (which = 0: lhs, 1: rhs)
 *                        into the plan's workspace (lhs digits negated for SUB);
 *   mhg_plan_pack_buffer device pointer and byte size of that packed operand -- plans
 *                        of equal geometry (same operand shape, q, op) share its layout;
 *   mhg_plan_gemm        the GEMM + epilogue on the current packs (no packing).
 * mhg_plan_run == pack(lhs) + pack(rhs) + gemm. */
mhg_status mhg_plan_pack(mhg_plan plan, int which, void *stream);
mhg_status mhg_plan_pack_buffer(mhg_plan plan, int which, void **ptr, uint64_t *bytes);
mhg_status mhg_plan_gemm(mhg_plan plan, void *stream);
mhg_status mhg_plan_counters(mhg_plan plan, mhg_counters *ctr);

/* Peer memory for the copy-engine panel exchange (multi-GPU, no reference
 * counterpart: the reference is single-process, multiply.hpp:25-29).  An owner
 * exports the device allocation holding a packed operand (mhg_plan_pack_buffer);
 * the other ranks of its row / column group map it once (same node, NVLink peer
 * access enabled lazily) and pull the bytes with mhg_copy_async, which runs on
 * the copy engines and leaves every SM to the GEMM.
 *   mhg_ipc_export  IPC handle of the allocation containing ptr, and ptr's offset in it
 *   mhg_ipc_open    map a peer's handle in this process; *base = the allocation's start
 *   mhg_ipc_close   unmap a base returned by mhg_ipc_open
 *   mhg_copy_async  cudaMemcpyAsync(dst, src, bytes, default direction) on stream */
typedef struct {
    unsigned char bytes[64];
} mhg_ipc_handle;
mhg_status mhg_ipc_export(const void *ptr, mhg_ipc_handle *handle, uint64_t *offset);
mhg_status mhg_ipc_open(const mhg_ipc_handle *handle, void **base);
mhg_status mhg_ipc_close(void *base);
mhg_status mhg_copy_async(void *dst, const void *src, uint64_t bytes, void *stream);
/* Kernel launches per run and the planner's description (tiles, chunks, limbs). */
mhg_status mhg_plan_info(mhg_plan plan, uint64_t *launches, uint64_t *tiles, uint32_t *limbs,
                         uint32_t *k_chunks, uint64_t *workspace_bytes);
/* The planner's kernel choice: unsigned_digits = 1 for u8 limb digits (long K: lower
 * power at the 1 kW cap), 0 for balanced s8 digits; cta_group = 1 (single-CTA k_gemm)
 * or 2 (CTA-pair k_gemm2). */
mhg_status mhg_plan_variant(mhg_plan plan, int *unsigned_digits, int *cta_group);
mhg_status mhg_plan_destroy(mhg_plan plan);

/* ---- plan sequences (TU/TURBO Schur sweeps) ----
 * A sequence of plans captured, in order, into ONE CUDA graph: mhg_sweep_run replays every
 * plan's packs and GEMM back to back with a single launch and no host work between the steps
 * (the Schur-update sweep of a block elimination: each step reads what the previous one
 * wrote, so the steps are serial on the device).  The plans must outlive the sweep, must not
 * be empty, and must not be in profiling mode when the sweep is created. */
typedef struct mhg_sweep_s *mhg_sweep;
mhg_status mhg_sweep_create(const mhg_plan *plans, uint32_t count, mhg_sweep *sweep);
mhg_status mhg_sweep_run(mhg_sweep sweep, void *stream);
/* Sum of the plans' scalar_macs (the reference's work counter over the whole sweep). */
mhg_status mhg_sweep_macs(mhg_sweep sweep, uint64_t *macs);
mhg_status mhg_sweep_destroy(mhg_sweep sweep);

/* ---- multi-GPU partition (one process per GPU) ----
 * C-stationary partition by top-level Morton blocks of the output: with P = 2^b ranks,
 * rank r owns the r-th contiguous 1/P slice of every container's flat store (a rectangle:
 * P = 2 halves, P = 4 quadrants, P = 8 n/4 x n/2 blocks) and updates only its own block
 * C[R_r, C_r] -- disjoint output rectangles are independent (multiply.hpp:25-29), so no
 * reduction is needed.  K is cut into mhg_dist_segment_count(P) segments; segment s needs
 * A[R_r, k0:k1] -- a contiguous flat range of ONE rank's slice (a_owner) -- and
 * B[k0:k1, C_r] -- the whole slice of ONE rank (b_owner).  The geometry calls are pure host
 * code (usable without a GPU); the communication belongs to the host program (NCCL / MPI /
 * peer copies): per segment the owner packs its part (mhg_plan_pack on the plan from
 * mhg_dist_plan_create), the packed bytes (mhg_plan_pack_buffer) are broadcast inside the
 * row group (A part) / column group (B part), and every rank runs mhg_plan_gemm.
 * paper_1705_04807_b200/dist.py is such a host program (one Python process per GPU). */
typedef struct {
    uint32_t rank;
    uint64_t i0, j0, rows, cols; /* the rank's block of every container */
    uint32_t row_band, col_band; /* ranks sharing row_band form its row group, likewise columns */
} mhg_dist_block_t;
typedef struct {
    uint32_t index;
    uint64_t k0, k1;           /* inner range of the segment */
    uint32_t a_owner;          /* rank holding A[R_r, k0:k1] */
    uint64_t a_begin, a_end;   /* its flat cell range (inside a_owner's slice) */
    uint32_t b_owner;          /* rank holding B[k0:k1, C_r] */
    uint64_t b_begin, b_end;   /* its flat cell range (b_owner's whole slice) */
} mhg_dist_segment_t;
mhg_status mhg_dist_block(uint32_t nranks, uint32_t rank, uint64_t n, uint64_t t, mhg_dist_block_t *block);
/* Flat [begin, end) of the rank's slice of an n x n store. */
mhg_status mhg_dist_slice(uint32_t nranks, uint32_t rank, uint64_t n, uint64_t *begin, uint64_t *end);
mhg_status mhg_dist_segment_count(uint32_t nranks, uint32_t *count);
mhg_status mhg_dist_segment(uint32_t nranks, uint32_t rank, uint64_t n, uint64_t t, uint32_t index,
                            mhg_dist_segment_t *segment);
/* The rank's plan of one K segment: C[R_r, C_r] op= A[R_r, k0:k1] * B[k0:k1, C_r] on three
 * full-size same-layout containers (out, lhs, rhs).  A SET update overwrites with segment 0
 * only; later segments accumulate (the plan of segment index > 0 is created with ADD). */
mhg_status mhg_dist_plan_create(mhg_matrix out, mhg_matrix lhs, mhg_matrix rhs, mhg_op op,
                                uint32_t nranks, uint32_t rank, uint32_t index, mhg_plan *plan);

/* ---- verification and seeded inputs ---- */
/* Freivalds check of a finished multiply on the device: out_new == out_old op lhs*rhs
 * (views of matching shapes; out_old holds the output's cells from before the call,
 * in its own container) is tested as  C_new r == C_old r op A (B r)  (mod q) for
 * `rounds` random vectors r derived from `seed`; a wrong result survives a round with
 * probability <= 1/q.  *ok = 1 when every round agrees.  The device analogue of the
 * reference's cross-check (MismatchError, bench.hpp:123-125, 186-193).  Synchronous. */
mhg_status mhg_verify(mhg_view out_new, mhg_view out_old, mhg_view lhs, mhg_view rhs, mhg_op op,
                      uint32_t rounds, uint64_t seed, int *ok, void *stream);
/* mh::Rng (bench.hpp:44-52): std::mt19937_64(seed), below(k) = (next() * k) >> 64.
 * mhg_rng_below writes `count` consecutive draws of below(k) (k <= 2^32) -- a
 * container filled in flat Morton order from one stream is the reference's
 * gen_problem fill (:101-103).  Host only. */
typedef struct mhg_rng_s *mhg_rng;
mhg_status mhg_rng_create(uint64_t seed, mhg_rng *out);
mhg_status mhg_rng_below(mhg_rng rng, uint64_t k, uint32_t *dst, uint64_t count);
mhg_status mhg_rng_destroy(mhg_rng rng);

/* ---- diagnostics for tests / bench ---- */
/* Host helper: the limb representation parameters the planner picks for q
 * (number of int8 limbs, representative threshold, max K per int32 chunk). */
mhg_status mhg_limb_params(uint32_t q, uint32_t *limbs, uint32_t *threshold, uint64_t *k_max);
/* Host helper: the fold level the 2-limb epilogue uses for chunks of k_chunk
 * inner products (1, 2 or 3 Barrett reductions per output; 3 when q needs more
 * or fewer than 2 limbs or 2^16 mod q >= 256).  See DESIGN.md "Fold levels". */
mhg_status mhg_fold_level(uint32_t q, uint64_t k_chunk, uint32_t *level);
/* The same for plans with unsigned (u8) digits (mhg_plan_variant). */
mhg_status mhg_fold_level_u8(uint32_t q, uint64_t k_chunk, uint32_t *level);
/* Times `iters` replays of a plan's GEMM kernel alone (CUDA events on
 * `stream`), returns the mean ms per launch in *ms. */
mhg_status mhg_plan_time_gemm(mhg_plan plan, int iters, void *stream, float *ms);
/* Profiling mode: while enabled, mhg_plan_run launches the three kernels
 * directly (no graph) and brackets the GEMM launch with CUDA events on
 * `stream`; mhg_plan_gemm_time synchronises, returns the summed GEMM time and
 * the number of GEMM launches recorded since the last call, and resets. */
mhg_status mhg_plan_set_profiling(mhg_plan plan, int enable);
mhg_status mhg_plan_gemm_time(mhg_plan plan, float *total_ms, uint64_t *launches);

#ifdef __cplusplus
}
#endif

#endif /* MHG_H */
