/*
 * btas_cuda.h — C ABI of libbtas_cuda.so, the B200 (sm_100a) tropical-algebra
 * kernels behind the drop-in `paper_1701_04733_b200` package.
 *
 * The reference (`btas`, /root/reference/pkg/src/btas) is pure Python/NumPy
 * and has no FFI: its replaceable boundary is the Python API of the hot-path
 * functions.  Each entry point below replaces the compute body of one
 * reference function (cited per declaration); the Python mirror in
 * paper_1701_04733_b200/ keeps the reference names, argument meaning and
 * exceptions and calls these through ctypes.
 *
 * Conventions (all entry points):
 *  - Plain pointers to DEVICE memory, 64-bit sizes / leading dimensions in
 *    elements, row-major storage.  No torch types cross this boundary.
 *  - Every call is stream-ordered on the caller's `stream` (a cudaStream_t;
 *    NULL = legacy default stream).  Calls never allocate device memory and
 *    never synchronise the host; scratch space is passed in as `workspace`.
 *  - Return value: BTAS_OK (0) or a BTAS_ERR_* status; the Python layer maps
 *    statuses to exceptions (btas_status_string gives the text).
 *  - Storage is "oriented" exactly like the reference (matrix.py:3-7,82-95):
 *    the symbolic Infinity is stored as +inf under min-plus and -inf under
 *    max-plus.  int32 storage encodes it as +/-BTAS_I32_INF and keeps finite
 *    entries strictly inside (-BTAS_I32_LIMIT, BTAS_I32_LIMIT).
 *  - dev_flags is an int32[BTAS_NUM_FLAGS] device array; kernels only ever
 *    OR bits into it (set-only, like the reference's saturation flag,
 *    semiring.py:73-88).
 */
#ifndef BTAS_CUDA_H
#define BTAS_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* btas_stream_t; /* == cudaStream_t */

/* element types of the storage */
enum { BTAS_F32 = 0, BTAS_I32 = 1, BTAS_F64 = 2 };
/* semiring kinds (reference SemiringKind, semiring.py:17-29) */
enum { BTAS_MIN_PLUS = 0, BTAS_MAX_PLUS = 1 };

/* int32 storage encoding of Infinity and the finite-domain limit */
#define BTAS_I32_INF 0x3FFFFFFF
#define BTAS_I32_LIMIT (1 << 28)

/* dev_flags slots */
enum {
  BTAS_FLAG_CHANGED = 0,   /* output differs from `Cprev` (fixpoint test, apsp.py:161) */
  BTAS_FLAG_DIAG_NEG = 1,  /* an output diagonal entry is < 0 (apsp.py:125,168,171) */
  BTAS_FLAG_SATURATED = 2, /* a finite (x) finite product saturated (matrix.py:334-342) */
  BTAS_FLAG_PATH = 3,      /* OR of (1 << path) for every GEMM path that ran (diagnostics) */
  BTAS_NUM_FLAGS = 8
};

/* btas_gemm_verify comparison modes (reference apsp.py:202-208) */
enum {
  BTAS_VERIFY_LE = 1, /* violation where !(Cref <= A (x) B): the triangle inequality d <= d (x) d */
  BTAS_VERIFY_EQ = 2  /* violation where A (x) B != Cref: the closure fixpoint d (x) (I (+) A) = d */
};

/* GEMM kernel paths (bit index in BTAS_FLAG_PATH) */
enum {
  BTAS_PATH_FAST32 = 0,  /* f32 FADD2+FMNMX3 / i32 VIADDMNMX */
  BTAS_PATH_S16X2 = 1,   /* integer operands with |x| < 2^12: VIADDMNMX.S16x2, 2 pairs/instr */
  BTAS_PATH_CHECKED = 2, /* per-candidate overflow masking (the reference's masked tile) */
  BTAS_PATH_FAST64 = 3,  /* f64 DADD + min */
  BTAS_PATH_EMPTY = 4,   /* no work (an operand has no rows/cols) */
  BTAS_PATH_I32F64 = 5   /* f64 integer operands whose sums stay inside the int32 domain: VIADDMNMX */
};

/* status codes */
enum {
  BTAS_OK = 0,
  BTAS_ERR_INVALID = 1,     /* bad argument (null pointer, negative size, bad dtype/kind) */
  BTAS_ERR_CUDA = 2,        /* a CUDA runtime call or launch failed */
  BTAS_ERR_WORKSPACE = 3,   /* workspace too small */
  BTAS_ERR_UNSUPPORTED = 4  /* combination not supported */
};

/* Statistics of one ingest/scan pass (written on the device, read by the host). */
typedef struct btas_stats {
  unsigned long long nan_count;      /* NaN entries (ingest: rejected, matrix.py:88-89) */
  unsigned long long neg_inf_count;  /* -inf in symbolic input (ingest: rejected, matrix.py:90-91) */
  unsigned long long non_integral;   /* finite entries with a fractional part */
  unsigned long long over_limit;     /* finite |x| >= the dtype's integer limit (matrix.py:98-115) */
  unsigned long long out_of_range;   /* finite input not representable in the target dtype */
  unsigned long long finite_count;   /* finite entries */
  unsigned long long max_abs_key;    /* ordered key of max |finite| (decode with btas_key_to_double) */
  unsigned long long min_key;        /* ordered key of min finite */
  unsigned long long max_key;        /* ordered key of max finite */
} btas_stats;

const char* btas_version(void);
const char* btas_status_string(int status);
/* decode an ordered key of btas_stats; returns NaN for the "no finite entry" key */
double btas_key_to_double(unsigned long long key);
/* Copy `words` 32-bit words (<= 4096) from device memory to `dst` with SM
 * stores, where dst may be page-locked host memory (cudaHostAlloc'd, mapped
 * under unified addressing).  The host reads small results (stats, flag words)
 * this way so the read never queues behind an unrelated bulk device->host copy
 * on the copy engine; the caller synchronises on an event after the call. */
int btas_export_words(const void* src, void* dst, int64_t words, btas_stream_t stream);
/* reset a device btas_stats before an ingest/scan */
int btas_stats_init(btas_stats* stats_dev, btas_stream_t stream);

/* Ingest symbolic-form values (f64 or f32 device array, +inf = Infinity) into
 * oriented storage of `dst_dtype`: validates (NaN, -inf), normalises -0.0,
 * orients Infinity per kind, encodes int32, and accumulates statistics.
 * Replaces TropicalMatrix/TropicalVector construction (matrix.py:82-115,132-156). */
int btas_ingest(int kind, int src_dtype, const void* src, int64_t numel,
                int dst_dtype, void* dst, btas_stats* stats_dev, btas_stream_t stream);

/* Statistics of oriented storage (max |finite|, min/max finite): the
 * saturation screens of matrix.py:297-312 and apsp.py:103-107. */
int btas_scan(int dtype, const void* x, int64_t numel, btas_stats* stats_dev, btas_stream_t stream);

/* Oriented storage -> oriented float64 (identical to the reference's .data). */
int btas_to_f64(int dtype, const void* src, int64_t numel, double* dst, btas_stream_t stream);

/* Fill with Infinity (oriented for kind) or a finite value.
 * TropicalMatrix.filled (matrix.py:158-168). */
int btas_fill(int dtype, int kind, void* x, int64_t numel, double value, btas_stream_t stream);

/* identity_matrix (matrix.py:257-263): 0 on the diagonal, Infinity elsewhere. */
int btas_identity(int dtype, int kind, void* d, int64_t ld, int64_t n, btas_stream_t stream);

/* _closure_base (apsp.py:80-90): dst = src with diag <- min(diag, 0). */
int btas_closure_base(int dtype, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t n,
                      btas_stream_t stream);

/* ew_add (matrix.py:271-277), for matrices and vectors: out = a (+) b elementwise. */
int btas_ewadd(int dtype, int kind, const void* a, const void* b, void* out, int64_t numel,
               btas_stream_t stream);

/* Tropical GEMM: C = (A (x) B) [(+) Z], with the reference's saturation
 * semantics.  Replaces matmul/_product_tile/_saturation_limit
 * (matrix.py:297-400).
 *   integer_mode : the operands are integer-valued (reference `integer`
 *                  flag); selects the integer saturation limit (2^53 f64,
 *                  2^24 f32, always 2^28 for i32) and allows the S16X2 path.
 *   Z, Cprev     : nullable.  Z is the accumulate_into operand (read only);
 *                  Cprev sets BTAS_FLAG_CHANGED when C != Cprev bytewise.
 *   C may alias Z but not A, B or Cprev.
 * The kernel path is chosen ON THE DEVICE by an exact screen over per-k
 * operand extremes, so the call never synchronises. */
size_t btas_gemm_workspace_bytes(int dtype, int64_t M, int64_t N, int64_t K);
int btas_gemm(int dtype, int kind, int integer_mode,
              const void* A, int64_t lda, const void* B, int64_t ldb,
              const void* Z, int64_t ldz, void* C, int64_t ldc,
              int64_t M, int64_t N, int64_t K,
              const void* Cprev, int64_t ldcp,
              int32_t* dev_flags, void* workspace, size_t workspace_bytes,
              btas_stream_t stream);

/* btas_gemm fused with an all-gather over peer memory: every element of C is
 * also stored at the same offset into peer_C[0..n_peers) (n_peers <= 7) —
 * the other ranks' buffers mapped into this process over NVLink (CUDA IPC /
 * symmetric memory) — from the GEMM epilogue, so the exchange of row-sharded
 * results overlaps the add-min work tile by tile (no separate collective).
 * Peer stores are made visible system-wide before the kernel completes.
 * Used by the row-sharded squaring step (apsp.py:159). */
int btas_gemm_peers(int dtype, int kind, int integer_mode,
                    const void* A, int64_t lda, const void* B, int64_t ldb,
                    void* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                    const void* Cprev, int64_t ldcp, void* const* peer_C, int n_peers,
                    int32_t* dev_flags, void* workspace, size_t workspace_bytes,
                    btas_stream_t stream);

/* The product A (x) B compared entry by entry with Cref in the GEMM
 * epilogue, without storing it (the verifier's two products,
 * find_apsp_violation apsp.py:202-208): *first_bad (caller-initialised to
 * ~0) receives the smallest row-major index i*N + j that violates `mode`
 * (atomicMin, so any tile order gives the reference's np.argmax answer) and
 * BTAS_FLAG_CHANGED is set when any does.  Saturation behaves as btas_gemm.
 * Min-plus only. */
int btas_gemm_verify(int dtype, int kind, int integer_mode,
                     const void* A, int64_t lda, const void* B, int64_t ldb,
                     const void* Cref, int64_t ldcr, int64_t M, int64_t N, int64_t K,
                     int mode, unsigned long long* first_bad,
                     int32_t* dev_flags, void* workspace, size_t workspace_bytes,
                     btas_stream_t stream);

/* Predecessor product for path reconstruction (extension; the reference has
 * none): idx[i,j] <- the smallest k attaining
 * min_k A[i,k] (x) B[k,j] (min-plus, storage arithmetic), or -1 where that
 * minimum is not finite, differs from Cref[i,j], or row0 + i == j.  With A =
 * the distance matrix, B = the adjacency with an infinite diagonal and Cref =
 * the distances, idx is the last hop of a shortest path (the predecessor
 * matrix).  Same workspace as btas_gemm (btas_gemm_workspace_bytes).
 * operand_bound >= max |finite entry| of A and of B (negative: unknown):
 * integer data (int32, or integer_mode) below 2^12 with K <= 65536 runs as
 * packed (value << 16 | k) keys through the VIADDMNMX kernel (one
 * instruction per candidate); otherwise compare-and-select per candidate. */
int btas_gemm_argmin(int dtype, int integer_mode, double operand_bound, const void* A, int64_t lda,
                     const void* B, int64_t ldb, const void* Cref, int64_t ldcr, int64_t M, int64_t N,
                     int64_t K, int64_t row0, int32_t* idx, int64_t ldi, void* workspace,
                     size_t workspace_bytes, btas_stream_t stream);

/* Elementwise half of find_apsp_violation (apsp.py:194-200) in one pass over
 * D and the adjacency A (n x n, same storage): first[0] <- smallest i with
 * D[i,i] != 0, first[1] <- smallest row-major index with !(D <= I (+) A)
 * (atomicMin; first[] caller-initialised to ~0). */
int btas_verify_base(int dtype, const void* D, int64_t ldd, const void* A, int64_t lda, int64_t n,
                     unsigned long long* first, btas_stream_t stream);

/* Measurement hooks (bench.py): when enabled, every btas_gemm brackets its
 * GEMM kernel launches (not the screen/packing) with CUDA events recorded on
 * the caller's stream; btas_gemm_timing_read synchronises on them and returns
 * the summed kernel time and the number of bracketed calls (then clears). */
int btas_gemm_timing(int enable);
int btas_gemm_timing_read(double* total_ms, int* count);

/* Batched tropical matvec: Out[b, i] = (+)_k A[i, k] (x) V[b, k] for b < batch.
 * Always masks overflow like matrix.py:403-425. */
int btas_matvec(int dtype, int kind, int integer_mode,
                const void* A, int64_t lda, int64_t M, int64_t K,
                const void* V, int64_t ldv, int64_t batch,
                void* Out, int64_t ldo, int32_t* dev_flags, btas_stream_t stream);

/* btas_matvec with a caller-known bound: abs_bound >= max|finite A| +
 * max|finite V| (e.g. from the btas_stats.max_abs_key of each operand's
 * ingest, which immutable operands keep).  When the bound proves that no
 * finite (x) finite candidate can overflow (below 2^28 for int32, the
 * integer limit in integer mode, the largest finite value otherwise) the
 * kernels skip the per-element magnitude screen of matrix.py:408-420's mask
 * (the result and the flag are the same: nothing can saturate).  A negative
 * or NaN abs_bound means "unknown" = btas_matvec. */
int btas_matvec_bounded(int dtype, int kind, int integer_mode,
                        const void* A, int64_t lda, int64_t M, int64_t K,
                        const void* V, int64_t ldv, int64_t batch,
                        void* Out, int64_t ldo, double abs_bound,
                        int32_t* dev_flags, btas_stream_t stream);

/* Blocked three-phase Floyd-Warshall, in place on D (n x n, min-plus),
 * bit-identical to the sequential k-round program of apsp.py:93-133
 * (snapshot panels keep each round's operands exactly as the reference sees
 * them).  `masked` selects the overflow-masking rounds (apsp.py:111-123) the
 * reference uses when its screen fails; `max_abs`/`min_finite` are the scan of
 * D used to choose the kernel path.  Sets BTAS_FLAG_SATURATED on masked
 * overflow and BTAS_FLAG_DIAG_NEG when a diagonal entry ends < 0. */
size_t btas_fw_workspace_bytes(int dtype, int64_t n);
int btas_fw(int dtype, int integer_mode, void* D, int64_t ld, int64_t n, int masked,
            double max_abs, double min_finite, int32_t* dev_flags,
            void* workspace, size_t workspace_bytes, btas_stream_t stream);

/* Row-sharded Floyd-Warshall for P processes (one per GPU) with lookahead
 * groups: the same per-round operands as btas_fw.  Each rank holds rows
 * [slab_r0, slab_r0 + slab_rows) of D (slab_r0 a multiple of 128) at D_slab.
 * Pivot blocks (b = 128 rows, 64 for float64) are processed in groups of
 * up to btas_fw_dist_group_size(dtype) consecutive blocks [kb0, kb0 +
 * group_blocks) that lie inside ONE rank's slab (its owner).  Per group the
 * host runs, in order:
 *   OWNER   on the owner: for each block of the group, the pending updates of
 *           the group's earlier blocks into its row / column panels, phase 1,
 *           the row panel and the column panel over the owner's rows,
 *   a broadcast of the owner's workspace bytes [bcast_offset, +bcast_bytes)
 *           to every rank (one NCCL broadcast per group; or fused: see
 *           btas_fw_dist_group_peers),
 *   REST    on every rank: a non-owner's column panels for each block of the
 *           group, then the update of the rank's rows by the whole group in
 *           one GEMM pass (K = group_blocks * b);
 * INIT once before the first group and DIAG once at the end.  `masked` and
 * `min_finite` must be the same on every rank (all-reduced scan of D).  One
 * exchange per group instead of per pivot block (replaces the reference
 * rounds of apsp.py:108-123, byte-identical for any P). */
enum {
  BTAS_FW_STAGE_INIT = 0,
  BTAS_FW_STAGE_DIAG = 4,
  BTAS_FW_STAGE_OWNER = 5,
  BTAS_FW_STAGE_REST = 6
};
int btas_fw_dist_group_size(int dtype);
size_t btas_fw_dist_workspace_bytes(int dtype, int64_t n, int64_t slab_rows, size_t* bcast_offset,
                                    size_t* bcast_bytes);
int btas_fw_dist_group(int dtype, int integer_mode, int stage, void* D_slab, int64_t ld, int64_t n,
                       int64_t slab_r0, int64_t slab_rows, int64_t kb0, int group_blocks, int masked,
                       double min_finite, int32_t* dev_flags, void* workspace, size_t workspace_bytes,
                       btas_stream_t stream);
/* btas_fw_dist_group with the broadcast fused into the OWNER stage: every
 * store the owner's kernels make into its broadcast region is repeated, at
 * the same offset, in peer_regions[0..n_peers) (n_peers <= 7): the other
 * ranks' broadcast regions (their workspace + bcast_offset) mapped into this
 * process (NVLink peer memory / CUDA IPC).  The caller replaces the
 * broadcast by a barrier that orders the peers' REST stage after this OWNER
 * stage, and alternates two workspaces by the parity of the group so the
 * next owner's stores never overwrite a region a peer is still reading.
 * Other stages ignore the peers. */
int btas_fw_dist_group_peers(int dtype, int integer_mode, int stage, void* D_slab, int64_t ld, int64_t n,
                             int64_t slab_r0, int64_t slab_rows, int64_t kb0, int group_blocks, int masked,
                             double min_finite, int32_t* dev_flags, void* workspace, size_t workspace_bytes,
                             void* const* peer_regions, int n_peers, btas_stream_t stream);

/* Diagonal test: sets BTAS_FLAG_DIAG_NEG if any d[i,i] < 0 (apsp.py:125,168). */
int btas_diag_negative(int dtype, const void* d, int64_t ld, int64_t n, int32_t* dev_flags,
                       btas_stream_t stream);

/* Register/shared-memory microbenchmark of the add-min instruction mixes
 * (the roofline denominator).  mix: 0 = f32 FADD2+FMNMX3, 1 = i32 VIADDMNMX,
 * 2 = s16x2 VIADDMNMX.S16x2, 3 = f64 DADD + ternary compare (DSETP + FSEL).  Writes pairs per SM clock and the effective
 * SM clock (MHz) of the run.  Synchronises (diagnostic only). */
int btas_probe_ceiling(int mix, double* pairs_per_clk_sm, double* sm_mhz, double* tpairs_per_s);

/* Repeated-squaring APSP (apsp.py:136-178) of a small graph in ONE
 * cooperative kernel: every squaring, its fixpoint compare, the uncounted
 * negative-cycle probe and the result copy run on the device with grid-wide
 * barriers between dependent steps (no per-step host round trip).  base is
 * the closure base I (+) A (min-plus storage, n x n, 2 <= n <=
 * BTAS_APSP_SMALL_MAX_N); out receives the distances.  dev_result (device
 * int32[4]): multiplications_performed, negative_cycle, saturated, fixpoint.
 * The saturation bit is also ORed into dev_flags.  Results are identical to
 * the btas_gemm-driven loop. */
#define BTAS_APSP_SMALL_MAX_N 1024
size_t btas_apsp_small_workspace_bytes(int dtype, int64_t n);
int btas_apsp_squaring_small(int dtype, int integer_mode, const void* base, int64_t ldb, int64_t n,
                             void* out, int64_t ldo, int32_t* dev_result, int32_t* dev_flags,
                             void* workspace, size_t workspace_bytes, btas_stream_t stream);

/* ---------------------------------------------------------------------------
 * On-device instance generator: replaces random_graph + graph_to_matrix
 * (reference graph_io.py:273-304, 158-165) for dense instances.
 *
 * The reference draws from ONE numpy PCG64 stream (XSL-RR 128/64, the
 * state after SeedSequence seeding is passed in as btas_pcg64): first one
 * uniform double per ordered off-diagonal pair in row-major order
 * (present iff (u >> 11) < p_threshold, p_threshold = ceil(p * 2^53)), then
 * one weight per present edge:
 *   BTAS_WEIGHTS_CONST    integers(low, low+1): no draws, weight = low
 *   BTAS_WEIGHTS_BOUNDED  integers(low, low+range+1): Lemire bounded draws on
 *                         the 32-bit-buffered stream (range < 2^32) or on the
 *                         64-bit stream (range >= 2^32), with numpy's rejection
 *   BTAS_WEIGHTS_UNIFORM  uniform(low, low+scale): low + scale * double
 * and builds the dense min-plus matrix (diagonal 0, absent edges +inf,
 * converted and validated exactly as btas_ingest does from float64).
 *
 * Three stream-ordered stages; the caller reads the edge count written by
 * stage 1 to size the draw buffer, and the accepted-draw count written by
 * stage 2 to decide whether another window of draws is needed (only bounded
 * draws reject).  Draw buffer elements: uint32 (range < 2^32), uint64
 * (range >= 2^32) or double (uniform).
 * ------------------------------------------------------------------------- */
typedef struct btas_pcg64 {
  uint64_t state_hi, state_lo, inc_hi, inc_lo;
} btas_pcg64;

enum { BTAS_WEIGHTS_CONST = 0, BTAS_WEIGHTS_BOUNDED = 1, BTAS_WEIGHTS_UNIFORM = 2 };

/* workspace of all three stages for an n-vertex instance */
size_t btas_graph_workspace_bytes(int64_t n);
/* stage 1 (random_graph presence draws): *dev_edges (device int64) = number of present pairs */
int btas_graph_presence(const btas_pcg64* rng, int64_t n, uint64_t p_threshold, void* workspace,
                        size_t workspace_bytes, int64_t* dev_edges, btas_stream_t stream);
/* stage 2 (weight draws): consumes the 64-bit stream units [unit0, unit0 + units) past the
 * presence doubles, appends accepted draws with rank < edges to draws[], and advances
 * *dev_accepted (device int64, 0 before the first window).  units <= n*(n-1) + 2^20. */
int btas_graph_draw(const btas_pcg64* rng, int64_t n, int weights_mode, uint64_t range, double low,
                    double scale, int64_t edges, uint64_t unit0, uint64_t units, void* draws,
                    void* workspace, size_t workspace_bytes, int64_t* dev_accepted, btas_stream_t stream);
/* stage 3 (graph_to_matrix): dense n x n min-plus storage of dtype into D (leading dim ld);
 * reuses stage 1's presence record and counts in the workspace (rng and p_threshold
 * must be stage 1's); stats as btas_ingest reports them. */
int btas_graph_fill(int dtype, const btas_pcg64* rng, int64_t n, uint64_t p_threshold, int weights_mode,
                    uint64_t range, int64_t low, const void* draws, void* D, int64_t ld,
                    const void* workspace, size_t workspace_bytes, btas_stats* stats_dev,
                    btas_stream_t stream);

/* graph_to_matrix of an explicit edge list (reference graph_io.py:158-165 with
 * the Graph normalisation of :64-83: duplicate (src, dst) keep the minimum
 * weight, -0.0 -> +0.0): D = +inf off the diagonal, 0 on it, then every edge
 * min-scattered (a negative self-loop lowers the diagonal).  dev_errors
 * (device int64[3]) receives the smallest failing edge index per class, or m
 * when none fails: [0] src/dst outside [0, n), [1] non-finite weight,
 * [2] weight not representable in dtype (int32: integral, |w| < 2^28).
 * Statistics of the result: btas_scan. */
int btas_edges_to_matrix(int dtype, int64_t n, const int64_t* src, const int64_t* dst, const double* weight,
                         int64_t m, void* D, int64_t ld, int64_t* dev_errors, btas_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* BTAS_CUDA_H */
