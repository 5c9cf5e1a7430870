/*
 * include/vjp.h — C ABI of the B200 (sm_100a) vjp library  libvjp_b200.so
 *
 * The library computes the reverse-mode return sweeps (vector-Jacobian
 * products, "vjp") of the bulk-parallel combinators of
 * arXiv 2202.10297:
 *
 *   vjp_scan             sec 5.2, P:1131-1236   (scan / prefix sum)
 *   vjp_reduce           sec 5.1, P:971-1087    (reduce; special cases + * min max)
 *   vjp_reduce_by_index  sec 5.1.2, P:1090-1126 (histogram / multi-reduce)
 *   vjp_scatter          sec 5.3
 *   vjp_scatter_forward / vjp_scatter_restore   sec 5.3
 *
 * "P:n" is line n of PAPER.md.  Every entry point takes the primal inputs, an
 * operator tag and the output adjoint, and writes the input adjoint(s) by the
 * paper's rules.  Readings of the paper where it is silent are listed in
 * DESIGN.md ("Readings"); the ones that change results are repeated here.
 *
 * CONVENTIONS (all entry points)
 *  - Every array argument is a DEVICE pointer (cudaMalloc / torch CUDA
 *    tensor) owned by the caller, unless stated otherwise.  The library never
 *    allocates device memory, never synchronises the host, and is stream
 *    ordered: all work is enqueued on `stream` (a cudaStream_t; NULL = the
 *    legacy default stream).  Calls on different streams with different
 *    workspaces may run concurrently.
 *  - Value arrays are f32 or f64 (`vjp_dtype`); index arrays are int32 or
 *    int64 (`vjp_itype`).  Every array base pointer must be 16-byte aligned
 *    (VJP_EALIGN otherwise): the kernels move tiles with TMA and 128-bit
 *    vector accesses.
 *  - Scan element layouts: ADD/MUL/MIN/MAX one scalar per element;
 *    LINREC two scalars (d, c) interleaved (AoS); MAT2 four scalars, a 2x2
 *    matrix row-major.  n always counts ELEMENTS, not scalars.
 *  - `ws` is a device workspace of at least the bytes returned by the matching
 *    *_workspace_bytes query (VJP_EWORKSPACE otherwise); it is overwritten
 *    (its header is cleared on `stream` inside the call) and may be reused
 *    by the next call on the same stream.  ws may be NULL iff the query
 *    returns 0.
 *  - flags: VJP_ACCUMULATE turns "as_bar = contribution" into the paper's
 *    "as_bar += contribution" (reading R6).  Without it,
 *    every element of the output adjoint is written.
 *  - Arguments are validated before anything is enqueued; an argument error
 *    returns non-zero and enqueues nothing.  A launch failure returns
 *    VJP_ECUDA (cudaGetLastError); asynchronous kernel faults surface at the
 *    caller's next synchronisation, as for any CUDA library.
 *  - n == 0 is a no-op (outputs untouched; an optional primal output gets
 *    the neutral element).
 *  - Arithmetic: f64 data is computed in f64; f32 data is loaded as f32 and
 *    computed/accumulated in f64, outputs rounded once to f32 (reading R9).
 *    Round-to-nearest-even, no flush-to-zero.
 *  - A call's behaviour depends only on its arguments.  Tuning environment
 *    variables (VJP_SWEEP_K / _D / _ROUND_MB, VJP_LB_L2_MB, VJP_LB_VARIANT,
 *    VJP_KMEANS_FFMA; testing only) are read ONCE per process at first use,
 *    never per call.
 */
#ifndef VJP_B200_H
#define VJP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *vjp_stream_t; /* identical to cudaStream_t */

typedef enum { VJP_F32 = 1, VJP_F64 = 2 } vjp_dtype;
typedef enum { VJP_I32 = 1, VJP_I64 = 2 } vjp_itype;

/* Operator tags (the associative (.) of scan / reduce / reduce_by_index).
 *  ADD, MUL, MIN, MAX : scalar +, *, min, max.
 *  LINREC : element (d, c); (d1,c1) (.) (d2,c2) = (d2 + c2*d1, c2*c1) — the
 *           paper's lin_o used as a primal operator (reading R2);
 *           ys_i = (D_i, C_i), D_i = c_i*D_{i-1} + d_i (first-order linear
 *           recurrence), C_i = prod c.  Neutral (0, 1).
 *  MAT2   : element a 2x2 matrix, R_i = R_{i-1} . A_i (scan order of P:1137,
 *           reading R1).  Neutral I. */
typedef enum {
    VJP_ADD = 1, VJP_MUL = 2, VJP_MIN = 3, VJP_MAX = 4, VJP_LINREC = 5, VJP_MAT2 = 6
} vjp_op;

typedef enum {
    VJP_OK = 0,
    VJP_EINVAL = 1,       /* bad argument (NULL where required, n < 0, m < 1, bad tag) */
    VJP_EUNSUPPORTED = 2, /* a tag/call with no rule in the paper or not built (see each call) */
    VJP_EWORKSPACE = 3,   /* ws_bytes smaller than the query */
    VJP_ECUDA = 4,        /* a CUDA launch / runtime call failed */
    VJP_EDUPINDEX = 5,    /* scatter: duplicate target (VJP_CHECK_INDICES only) */
    VJP_EOOB = 6,         /* index out of range (VJP_CHECK_INDICES only) */
    VJP_EALIGN = 7        /* an array base pointer is not 16-byte aligned */
} vjp_status;

enum {
    VJP_ACCUMULATE = 1u,     /* as_bar += contribution instead of = */
    VJP_CHECK_INDICES = 2u,  /* scatter: detect duplicates / out-of-range (synchronises) */
    VJP_SCAN_LOOKBACK = 1u << 16, /* tuning/testing: vjp_scan uses the single-sweep decoupled
                                    look-back kernels instead of the chunked reduce-then-scan
                                    kernels (MIN/MAX always use look-back) */
    VJP_SCAN_SWEEP = 1u << 17,    /* single GPU: the one-read L2-round sweep (one persistent
                                    kernel, as/ys_bar read from HBM once, each round re-read
                                    from L2) for any of ADD/MUL/LINREC/MAT2; the default for
                                    f64 ADD with ACCUMULATE.  The default for
                                    f64/f32 ADD without ys / ACCUMULATE is the one-pass kernel
                                    with a two-level decoupled look-back */
    VJP_SCAN_CHUNKED = 1u << 18,  /* tuning/testing: force the two chunked kernels (the default for
                                    MUL/LINREC/MAT2, and for ADD with ys or on several GPUs) */
    VJP_SCAN_BLOCKLB = 1u << 19   /* tuning/testing: force the one-read block look-back
                                    (single GPU, no ACCUMULATE; opt-in: measured slower than
                                    the chunked kernels) */
};

/* One shard of a multi-GPU call: this process owns global elements
 * [global_offset, global_offset + n_local) of a length-global_n problem,
 * shards are contiguous and ordered by rank.  world == 1 means no sharding. */
typedef struct {
    int32_t rank;
    int32_t world;
    int64_t global_offset;
    int64_t global_n;
} vjp_shard;

const char *vjp_status_string(vjp_status s);

/* Number of kernels this library has launched in this process so far (the
 * bench's gpu_launches count).  Host-side counter, thread-safe. */
uint64_t vjp_launch_count(void);

/* ======================================================================
 * vjp_scan — sec 5.2
 *
 * Primal: ys = scan (.) e as, ys_i = as_0 (.) ... (.) as_i.
 * Computes as_bar = ys_bar . J_scan(as).  The paper's rule: the
 * forward sweep re-executes the primal scan; the return sweep builds
 * per-element Jacobian pairs and runs a reverse scan with linear-function
 * composition (lin_o; generalised to d-vectors with (0, I) as
 * neutral), then a map.  Closed form for ADD:
 * as_bar = reverse (scan (+) (reverse ys_bar)), in which case
 * `as` is not read and may be NULL.
 *
 *   op      ADD, MUL, MIN, MAX, LINREC, MAT2.  MIN/MAX use the pick-left
 *           subgradient on ties (reading R3).
 *   dtype   VJP_F32 or VJP_F64, for as, ys_bar, as_bar, ys alike.
 *   n       elements (>= 0).
 *   as      [n x width] primal input (NULL allowed for ADD when ys == NULL).
 *   ys_bar  [n x width] output adjoint.
 *   as_bar  [n x width] input adjoint (output).  Must not alias as/ys_bar.
 *   ys      nullable [n x width]: receives the primal scan (recomputed in the
 *           return sweep, never stored as a tape).
 *   ws      workspace, >= vjp_scan_workspace_bytes(op, dtype, n).
 * Errors: VJP_EINVAL, VJP_EALIGN, VJP_EWORKSPACE, VJP_ECUDA.
 * ==================================================================== */
size_t vjp_scan_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n);
vjp_status vjp_scan(vjp_op op, vjp_dtype dtype, int64_t n, const void *as,
                    const void *ys_bar, void *as_bar, void *ys, void *ws, size_t ws_bytes,
                    vjp_stream_t stream, unsigned flags);

/* Multi-GPU phase split of vjp_scan (contiguous shards):
 *   1. vjp_scan_partial: forward re-execution over the local shard; writes
 *      this shard's partial record (forward aggregate of as; for world > 1
 *      also the reverse-map aggregate, which reads ys_bar) to `partial`
 *      (device, vjp_scan_partial_bytes(op, dtype) bytes).
 *   2. the caller all-gathers the records of all ranks, in rank order, into
 *      `gathered` (device, world x partial bytes) — e.g. NCCL all_gather.
 *   3. vjp_scan_finish: return sweep over the local shard, with this shard's
 *      forward carry (ranks < rank) and reverse carry (ranks > rank) combined
 *      from `gathered` on the device.
 * `n` is the LOCAL element count; `ws` must be the same workspace for both
 * phases (the finish reads the partial's per-tile prefixes).  MIN/MAX need a
 * second exchange (their reverse coefficients depend on the forward carry):
 * vjp_scan_partial2 below.  vjp_scan == partial + finish with world = 1.
 * An empty shard (n == 0) writes the neutral record. */
size_t vjp_scan_partial_bytes(vjp_op op, vjp_dtype dtype);
vjp_status vjp_scan_partial(vjp_op op, vjp_dtype dtype, int64_t n, const void *as,
                            const void *ys_bar, void *ws, size_t ws_bytes,
                            const vjp_shard *shard, void *partial, vjp_stream_t stream,
                            unsigned flags);
/* MIN/MAX scans need TWO exchanges (their reverse maps depend on the forward
 * carry): vjp_scan_partial (forward aggregate of the shard) ->
 * all_gather -> vjp_scan_partial2 (forward prefixes with the shard's forward
 * carry from gathered1, reverse-map aggregate of the shard -> partial2) ->
 * all_gather -> vjp_scan_finish with the second gathered array.  Other
 * operators: VJP_EUNSUPPORTED (one exchange suffices). */
vjp_status vjp_scan_partial2(vjp_op op, vjp_dtype dtype, int64_t n, const void *as,
                             const void *ys_bar, void *ws, size_t ws_bytes, const vjp_shard *shard,
                             const void *gathered1, void *partial2, vjp_stream_t stream,
                             unsigned flags);
vjp_status vjp_scan_finish(vjp_op op, vjp_dtype dtype, int64_t n, const void *as,
                           const void *ys_bar, void *as_bar, void *ys, void *ws,
                           size_t ws_bytes, const vjp_shard *shard, const void *gathered,
                           vjp_stream_t stream, unsigned flags);

/* ======================================================================
 * vjp_scan_cyclic — BLOCK-CYCLIC multi-GPU vjp_scan with a cross-GPU
 * decoupled look-back (the return sweep is a
 * scan with the associative lin_o, so its superblock aggregates compose).
 *
 * The global array of global_n elements is cut into superblocks (SB) of
 * sb_elems elements (the last one ragged).  SB J belongs to rank J % world;
 * a rank's LOCAL arrays (as, ys_bar, as_bar) hold its SBs J = rank, rank +
 * world, ... concatenated in increasing J (vjp_scan_cyclic_local_n elements).
 * Every rank runs ONE persistent sweep over its SBs from right to left, one
 * SB per round: all CTAs stream the SB once from HBM (the method bytes — no
 * pre-pass over ys_bar, unlike the contiguous split), compose the SB's
 * reverse map M_J, and CTA 0 pushes it (AGG) into EVERY rank's status buffer
 * over NVLink (peer-mapped stores, sys-scope release).  The carry entering
 * SB J is X_J = M_{J+1} o ... o M_{J+world-1} (E_{J+world}): the maps of the
 * other ranks' superblocks between J and this rank's previous superblock,
 * applied to the carry leaving that superblock, which the rank already holds
 * — so each rank waits only for the other ranks' AGG words (a look-back
 * terminated locally; no chain of inclusive carries across GPUs).  The CTAs
 * then apply the SB from L2 with X_J.  No collective on the ys_bar path.
 * For MUL / LINREC / MAT2 the forward re-execution needs each SB's forward
 * prefix: vjp_scan_cyclic_forward writes this rank's per-SB forward
 * aggregates (reads `as` once), the caller all-gathers them (world x
 * vjp_scan_cyclic_fwd_bytes, rank order) and passes the result as
 * `gathered` (ADD: neither call nor gathered is needed).
 *
 *   status[q]  rank q's status buffer (vjp_scan_cyclic_status_bytes), mapped
 *              into this process (torch symmetric memory / cudaIpc); zeroed
 *              once at allocation.  Word 0 of a rank's own buffer is set
 *              non-zero if one of its look-back waits timed out (a missing
 *              peer): the results of that call are then invalid.  Words
 *              1..8 hold the epoch each rank entered last: a call's first
 *              status write waits until every rank owning a superblock has
 *              entered its epoch (an in-kernel entry barrier, so one rank
 *              can never overwrite words another is still reading).
 *   epoch      1 .. 2^30-1, equal on all ranks for one call and STRICTLY
 *              INCREASING from call to call on the same status buffers (the
 *              status words carry it, so they are never reset).
 *   grid_ctas  0: the whole device, one cooperatively launched wave; > 0:
 *              that many CTAs (several virtual ranks sharing one device in
 *              tests — the caller keeps all ranks' CTAs co-resident).
 * All ranks must run the call concurrently (a rank's sweep waits on its
 * right neighbours' superblocks).  Errors: VJP_EINVAL (descriptor, sizes,
 * sb_elems not a multiple of vjp_scan_cyclic_tile_elems, or too large for
 * the grid: more than 8 tiles per CTA), VJP_EUNSUPPORTED (MIN/MAX: their
 * reverse maps need the forward carry), VJP_EWORKSPACE (vjp_scan_workspace_
 * bytes(op, dtype, n_local)), VJP_ECUDA.  Flags: VJP_ACCUMULATE.
 * ==================================================================== */
#define VJP_CYCLIC_MAX_RANKS 8
typedef struct {
    int32_t rank, world;
    int64_t global_n;   /* elements of the whole problem */
    int64_t sb_elems;   /* superblock elements (same on every rank) */
    uint32_t epoch;
    int32_t grid_ctas;
    void *status[VJP_CYCLIC_MAX_RANKS];  /* [world] peer-mapped DEVICE pointers */
} vjp_cyclic;
int64_t vjp_scan_cyclic_tile_elems(vjp_op op, vjp_dtype dtype);
int64_t vjp_scan_cyclic_sb_elems(vjp_op op, vjp_dtype dtype); /* suggested SB size for this device */
int64_t vjp_scan_cyclic_local_n(const vjp_cyclic *cy);
size_t vjp_scan_cyclic_status_bytes(vjp_op op, int64_t global_n, int64_t sb_elems);
size_t vjp_scan_cyclic_fwd_bytes(vjp_op op, vjp_dtype dtype, const vjp_cyclic *cy);
vjp_status vjp_scan_cyclic_forward(vjp_op op, vjp_dtype dtype, int64_t n_local, const void *as, void *ws,
                                   size_t ws_bytes, const vjp_cyclic *cy, void *sbagg, vjp_stream_t stream);
vjp_status vjp_scan_cyclic(vjp_op op, vjp_dtype dtype, int64_t n_local, const void *as, const void *ys_bar,
                           void *as_bar, void *ws, size_t ws_bytes, const vjp_cyclic *cy, const void *gathered,
                           vjp_stream_t stream, unsigned flags);

/* Host-side (CPU, no device) evaluation of the carry combination that
 * vjp_scan_finish performs on the device, for testing the multi-GPU logic
 * without a GPU.  gathered: HOST, world x partial records.  Writes this
 * rank's forward carry (width doubles) and reverse carry (width doubles). */
vjp_status vjp_scan_carries_host(vjp_op op, vjp_dtype dtype, int32_t rank, int32_t world,
                                 const void *gathered, double *fwd_carry, double *rev_carry);

/* ======================================================================
 * vjp_reduce — sec 5.1
 *
 * Primal: y = reduce (.) e as = as_0 (.) ... (.) as_{n-1}.
 *   ADD : as_bar_i = y_bar; forward not needed unless y/arg asked.
 *   MUL : forward computes (p = product of the nonzero elements [f64],
 *         z = number of zeros, i0 = first zero index) by a map-reduce
 *         (P:1055-1058); return: z = 0 -> as_bar_i = y_bar * p / as_i;
 *         z = 1 -> as_bar_{i0} = y_bar * p (reading R8: P:1051's "y" is the
 *         product of the nonzeros), 0 elsewhere; z >= 2 -> 0.
 *         -0.0 counts as a zero (IEEE compare).
 *   MIN/MAX : forward computes (y, i_y), i_y the FIRST index of the extremum
 *         (IEEE compare so -0.0 ties +0.0); return
 *         as_bar = 0 except as_bar[i_y] = y_bar.  With
 *         VJP_ACCUMULATE only as_bar[i_y] is touched (the paper's sparse
 *         adjoint).
 *   y_bar  DEVICE pointer to one element of dtype.
 *   as_bar [n] output.
 *   y      nullable DEVICE [1]: primal result (MUL: 0 if z > 0, else p).
 *   arg    nullable DEVICE int64[1]: i_y (MIN/MAX), i0 or -1 (MUL), -1 (ADD).
 *   LINREC / MAT2 : the paper's GENERAL reduce rule: y_bar is
 *         one element (W scalars) and as_bar_i = J_R^T (l_i, a_i) applied to
 *         the reverse product of the elements right of i — computed as the
 *         scan's return sweep seeded only at the last element (scan-last ==
 *         reduce) with a virtual ys_bar; y (nullable) = the reduction.
 * Errors: VJP_EINVAL, VJP_EALIGN, VJP_EWORKSPACE, VJP_ECUDA.
 * ==================================================================== */
size_t vjp_reduce_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n);
vjp_status vjp_reduce(vjp_op op, vjp_dtype dtype, int64_t n, const void *as,
                      const void *y_bar, void *as_bar, void *y, int64_t *arg, void *ws,
                      size_t ws_bytes, vjp_stream_t stream, unsigned flags);

/* Multi-GPU split: partial writes the shard's forward record (32 bytes:
 * MUL {double p; int64 z; int64 i0_global; pad}, MIN/MAX {double v; int64
 * i_global; ...}, ADD {double sum; ...}) to `partial` (device); the caller
 * all-gathers world records in rank order; finish combines them on the device
 * in rank order (deterministic) and runs the return map on the local shard. */
size_t vjp_reduce_partial_bytes(void);
vjp_status vjp_reduce_partial(vjp_op op, vjp_dtype dtype, int64_t n, const void *as, void *ws,
                              size_t ws_bytes, const vjp_shard *shard, void *partial,
                              vjp_stream_t stream);
vjp_status vjp_reduce_finish(vjp_op op, vjp_dtype dtype, int64_t n, const void *as,
                             const void *y_bar, void *as_bar, void *y, int64_t *arg, void *ws,
                             size_t ws_bytes, const vjp_shard *shard, const void *gathered,
                             vjp_stream_t stream, unsigned flags);

/* ======================================================================
 * vjp_reduce_by_index — sec 5.1.2
 *
 * Primal: hs = replicate m e; for i: hs[inds[i]] (.)= as[i];
 * bins outside [0, m) are skipped and get adjoint 0 (reading R4).  Return
 * sweep: the reduce rule with y_bar replaced by hs_bar[inds[i]]:
 *   ADD : as_bar_i = hs_bar[b_i] (a gather; `as` may be NULL).
 *   MUL : per-bin (p_b, z_b) forward histogram, then the three cases of
 *         vjp_reduce per bin.  p_b is accumulated as an exact integer sum of
 *         64-bit fixed-point log2|a| codes (sign folded in; DESIGN 7.4), so
 *         it does not depend on the order of the additions; relative error
 *         <= 0.7 * 2^-52 * (factors in the bin).
 *   MIN/MAX : per-bin winner (value, lowest index), as_bar = 0 except
 *         as_bar[winner_b] = hs_bar[b] (ACCUMULATE: only the winners).
 * VECTORISED operators (width > 1, "elementwise", reading A24):
 * element i is the row as[i][0..width), bin b the row hs[b][0..width); every
 * rule applies per component j — (b, j) has its own (p, z) and its own
 * lowest-index winner.  width = 1 is the hot path (config 4).
 * The general operator ("work is in progress") and LINREC/MAT2
 * return VJP_EUNSUPPORTED (see vjp_reduce_by_index_general for MUL).
 *   inds   [n] int32/int64 bins;  as [n x width];  hs_bar [m x width];
 *   as_bar [n x width] output.
 *   hs     nullable DEVICE [m x width]: primal histogram (ADD: the sum —
 *          DETERMINISTIC (stable bin sort + in-order segmented row sums,
 *          the routine vjp_kmeans accumulates its centers with) when ws
 *          holds vjp_reduce_by_index_hs_workspace_bytes (m <= 12287,
 *          n < 2^31), else by atomic adds (rounding order-dependent); MUL:
 *          product; MIN/MAX: extremum, +-inf for an empty (bin, component)).
 *   winners nullable DEVICE int64[m x width]: MIN/MAX winner ELEMENT index
 *          (-1 empty), MUL: zero count, ADD: -1.
 * Errors: VJP_EINVAL (width < 1, m < 1, NULL inputs), VJP_EUNSUPPORTED
 * (LINREC/MAT2), VJP_EALIGN, VJP_EWORKSPACE, VJP_ECUDA.
 * ==================================================================== */
size_t vjp_reduce_by_index_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n, int64_t m, int64_t width);
size_t vjp_reduce_by_index_hs_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n, int64_t m, int64_t width);
vjp_status vjp_reduce_by_index(vjp_op op, vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m, int64_t width,
                               const void *inds, const void *as, const void *hs_bar,
                               void *as_bar, void *hs, int64_t *winners, void *ws,
                               size_t ws_bytes, vjp_stream_t stream, unsigned flags);

/* vjp_reduce_by_index_general — the paper's GENERAL rule for reduce_by_index
 * (sec 5.1.2: "radix sort + segmented scans", left "work in
 * progress" there), for MUL: per bin b, as_bar_i (+)= hs_bar[b] * l_i * r_i
 * with l_i / r_i the product of the bin's other elements before / after i
 * (the reduce rule of P:986-1013 per bin).  Counting sort by bin, then one
 * warp per bin runs the forward and backward exclusive product scans.  Same
 * arguments as vjp_reduce_by_index without the primal outputs; op must be
 * VJP_MUL (ADD / MIN / MAX: VJP_EUNSUPPORTED — their special cases ARE the
 * general rule); flags: VJP_ACCUMULATE only.  Domain: the partial products
 * stay finite and normal (the special-case path tracks exponents instead).
 * Out-of-range bins: as_bar 0 (R4).  Workspace (n + m) * 24 bytes-ish, from
 * the query.  Results equal vjp_reduce_by_index(VJP_MUL) up to rounding. */
size_t vjp_reduce_by_index_general_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n, int64_t m);
vjp_status vjp_reduce_by_index_general(vjp_op op, vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m,
                                       const void *inds, const void *as, const void *hs_bar,
                                       void *as_bar, void *ws, size_t ws_bytes, vjp_stream_t stream,
                                       unsigned flags);

/* Multi-GPU split (partition by input range; per-bin state all-reduced;
 * width 1; the workspace is vjp_reduce_by_index_workspace_bytes(.., 1)):
 *   partial: per-bin state of the local shard into bin_val (DEVICE, 8 bytes
 *            per bin) and bin_aux (DEVICE int64[m]):
 *              MUL     bin_val = int64 code sum of the shard's nonzero factors
 *                      (bit pattern stored in the 8-byte slot; code(a) =
 *                      round(log2|a| 2^51) + [a < 0] 2^63 mod 2^64, DESIGN 7.4),
 *                      bin_aux = zero count
 *                      -> all_reduce SUM over int64 of both (exact: integer
 *                         adds mod 2^64, independent of order and of world)
 *              MIN/MAX bin_val = local extremum (+-inf if empty), bin_aux =
 *                      lowest GLOBAL index reaching it (INT64_MAX if empty)
 *                      -> all_reduce MIN/MAX(bin_val), then
 *                         vjp_reduce_by_index_select, then all_reduce MIN(bin_aux)
 *              ADD     nothing to exchange (returns immediately)
 *   select : MIN/MAX only: bin_aux[b] = INT64_MAX where the local extremum is
 *            not the global one (bin_val now holds the global value).
 *   finish : return sweep over the local shard from the combined state.
 * Shards use shard->global_offset to form global indices. */
vjp_status vjp_reduce_by_index_partial(vjp_op op, vjp_dtype dtype, vjp_itype itype, int64_t n,
                                       int64_t m, const void *inds, const void *as, void *ws,
                                       size_t ws_bytes, const vjp_shard *shard, double *bin_val,
                                       int64_t *bin_aux, vjp_stream_t stream);
vjp_status vjp_reduce_by_index_select(vjp_op op, int64_t m, const double *bin_val_global,
                                      const double *bin_val_local, int64_t *bin_aux,
                                      vjp_stream_t stream);
vjp_status vjp_reduce_by_index_finish(vjp_op op, vjp_dtype dtype, vjp_itype itype, int64_t n,
                                      int64_t m, const void *inds, const void *as,
                                      const void *hs_bar, void *as_bar, const double *bin_val,
                                      const int64_t *bin_aux, void *ws, size_t ws_bytes,
                                      const vjp_shard *shard, vjp_stream_t stream, unsigned flags);

/* ======================================================================
 * vjp_scatter — sec 5.3
 *
 * Primal: ys = scatter xs is vs: ys = xs except ys[is[j]] = vs[j]
 * (P:1241-1244); `is` must hold no duplicate in-range target.
 * Return sweep:
 *     vs_bar += gather is ys_bar        (vs_bar[j] = ys_bar[is[j]])
 *     xs_bar  = scatter ys_bar is (replicate m 0)
 * Elements are `width` scalars (width >= 1).  Out-of-range targets are
 * skipped and their vs_bar is 0 (reading R4).  xs_bar MAY alias ys_bar: then
 * the call is in place and its work is O(m), independent of n;
 * otherwise ys_bar is first copied to xs_bar (O(n)).  The paper's step (3),
 * restoring the primal xs, is not part of the adjoint: vjp_scatter_restore
 * (below) does it.
 *   is [m] int32/int64; ys_bar [n x width]; xs_bar [n x width]; vs_bar [m x width].
 * VJP_CHECK_INDICES: validates `is` first (synchronises the stream) and
 * returns VJP_EDUPINDEX / VJP_EOOB without touching the outputs; it needs a
 * workspace of vjp_scatter_workspace_bytes (a bitmap of n bits); without it
 * ws may be NULL.  VJP_ACCUMULATE applies to vs_bar (the paper's +=); xs_bar
 * is always the assignment of P:1275.
 * ==================================================================== */
size_t vjp_scatter_workspace_bytes(vjp_dtype dtype, int64_t n, int64_t m);
vjp_status vjp_scatter(vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m, int64_t width,
                       const void *is, const void *ys_bar, void *xs_bar, void *vs_bar, void *ws,
                       size_t ws_bytes, vjp_stream_t stream, unsigned flags);

/* vjp_scatter_shard — multi-GPU split of vjp_scatter (sec 5.3): ys_bar is
 * partitioned contiguously, this rank owns global elements [global_offset,
 * global_offset + n_local); `is` holds the m GLOBAL targets (replicated).
 * The call zeroes the owned targets of xs_bar (in place when xs_bar aliases
 * ys_bar: O(m)) and writes vs_bar_partial[j] = ys_bar[is[j] - global_offset]
 * for owned targets, 0 otherwise; the caller SUMs vs_bar_partial over the
 * ranks (exactly one rank owns each in-range target, so the sum is exact) —
 * one all_reduce of m * width scalars (paper_2202_10297_b200.dist.scatter).
 * No flags (accumulate / index checks are the caller's, after the sum). */
vjp_status vjp_scatter_shard(vjp_dtype dtype, vjp_itype itype, int64_t n_local, int64_t m, int64_t width,
                             const void *is, const void *ys_bar, void *xs_bar, void *vs_bar_partial,
                             const vjp_shard *shard, vjp_stream_t stream);

/* ======================================================================
 * vjp_scatter_forward / vjp_scatter_restore — the in-place scatter's forward
 * save and the return sweep's step (3) (sec 5.3)
 *
 * The in-place update `let xs = scatter xs is vs` overwrites xs, so the
 * forward sweep first saves the elements about to be overwritten:
 *     xs_saved = gather xs is;  xs = scatter xs is vs
 * and the return sweep, after vjp_scatter, restores the primal:
 *     xs = scatter ys is xs_saved
 * vjp_scatter_forward: xs [n x width] is updated IN PLACE (it becomes ys);
 *   xs_saved [m x width] is written (out-of-range targets: skipped, saved 0,
 *   reading R4); vs [m x width] is read.
 * vjp_scatter_restore: ys [n x width] is updated IN PLACE (it becomes xs
 *   again) from xs_saved; out-of-range targets are skipped.
 * Both are O(m): one thread per (target, component), nothing proportional to
 * n is touched.  DEVICE pointers, 16-byte aligned; `is` must hold no
 * duplicate in-range target — with VJP_CHECK_INDICES (forward
 * only; needs vjp_scatter_workspace_bytes of ws, synchronises) a violation
 * returns VJP_EDUPINDEX / VJP_EOOB before anything is written.  flags other
 * than VJP_CHECK_INDICES are rejected (VJP_EINVAL).
 * ==================================================================== */
vjp_status vjp_scatter_forward(vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m, int64_t width,
                               const void *is, const void *vs, void *xs, void *xs_saved, void *ws,
                               size_t ws_bytes, vjp_stream_t stream, unsigned flags);
vjp_status vjp_scatter_restore(vjp_dtype dtype, vjp_itype itype, int64_t n, int64_t m, int64_t width,
                               const void *is, const void *xs_saved, void *ys, vjp_stream_t stream);

/* Test hook: code[i] = the 64-bit factor code the MUL histograms accumulate
 * (reduce_by_index, DESIGN 7.4): round(log2|x[i]| 2^51) + [x[i] < 0] 2^63
 * mod 2^64, as computed by the kernels (x finite, nonzero; DEVICE arrays). */
vjp_status vjp_debug_mul_code(const double *x, int64_t *code, int64_t n, vjp_stream_t stream);

/* ======================================================================
 * vjp_scan_batched — vjp of a VECTORISED scan
 *
 * ys = scan (map (.)) e xs over n elements of `width` components each; the
 * paper's transpose rule makes it `width` independent scans
 * along n, component j of element i at [i][j] (each component Op::W scalars:
 * 1 for ADD/MUL, (d, c) for LINREC, a row-major 2x2 for MAT2).  The return
 * sweep is computed per component exactly as vjp_scan (the vectorised plus
 * case, is the per-column reversed suffix sum).
 *   as [n][width][W] (NULL allowed for ADD); ys_bar, as_bar likewise.
 * VJP_ACCUMULATE: as_bar += .  MIN/MAX (pick-left subgradient) take two more
 * passes (their reverse maps need the forward carry).  Errors: VJP_EINVAL,
 * VJP_EALIGN, VJP_EWORKSPACE, VJP_ECUDA.
 * ==================================================================== */
size_t vjp_scan_batched_workspace_bytes(vjp_op op, vjp_dtype dtype, int64_t n, int64_t width);
vjp_status vjp_scan_batched(vjp_op op, vjp_dtype dtype, int64_t n, int64_t width, const void *as,
                            const void *ys_bar, void *as_bar, void *ws, size_t ws_bytes,
                            vjp_stream_t stream, unsigned flags);

/* ======================================================================
 * vjp_kmeans — composite k-means cost gradient (BASELINE
 * config 5)
 *
 * f(C) = sum_p min_j ||p - c_j||^2 (reading R15: squared distance; ties go
 * to the FIRST center).  One call runs the forward (distances,
 * argmin, cost) and the return sweep with cost_bar = ybar:
 *   centers_bar[j] = 2 ybar sum_{p: a(p) = j} (c_j - p)
 * — the sum's adjoint, the min's sparse adjoint (only the
 * argmin's distance receives ybar) and the distance map's vjp,
 * accumulated per center as a width-d reduce_by_index(+) into k bins
 * (done as a stable counting sort + in-order segmented sum, so
 * the result is deterministic) — and the jvp of that vjp in the all-ones
 * direction, the Hessian diagonal hess_diag[j][t] = 2 ybar cnt_j.
 *   points  [n x d] row-major, centers [k x d]; f32 or f64 (arithmetic f64).
 *   cost_bar DEVICE [1].  centers_bar [k x d] output.
 *   hess_diag, assign (int32 [n]), counts (int64 [k]), cost ([1]): nullable
 *   DEVICE outputs.  VJP_ACCUMULATE adds into centers_bar, hess_diag, counts
 *   and cost (per-shard partials of a multi-GPU run are sums over points).
 * Limits: n < 2^31, 1 <= k <= 12288 (VJP_EUNSUPPORTED beyond), d >= 1.
 * Errors: VJP_EINVAL, VJP_EALIGN (element misalignment), VJP_EWORKSPACE,
 * VJP_ECUDA.  The workspace holds per-center/per-block tables and two int32
 * arrays of n (point order, assignment when `assign` is NULL).
 * ==================================================================== */
size_t vjp_kmeans_workspace_bytes(vjp_dtype dtype, int64_t n, int64_t k, int64_t d);
vjp_status vjp_kmeans(vjp_dtype dtype, int64_t n, int64_t k, int64_t d, const void *points,
                      const void *centers, const void *cost_bar, void *centers_bar, void *hess_diag,
                      int32_t *assign, int64_t *counts, void *cost, void *ws, size_t ws_bytes,
                      vjp_stream_t stream, unsigned flags);

/* ======================================================================
 * Calibration (measurement only, no vjp): the L2 ceilings the m = 10^6
 * reduce_by_index kernels are compared against (DESIGN 7.4, bench.py
 * --workload rbi): n random 8-byte gathers (vjp_calib_l2_gather, out: one
 * partial sum per thread, vjp_calib_out_len() doubles) or f64 red.adds
 * (vjp_calib_l2_red) into an L2-resident table, bins int32 read by 128-bit
 * loads as the histogram kernels do.  n % 4 == 0; idx entries in range.
 * ==================================================================== */
int64_t vjp_calib_out_len(void);
vjp_status vjp_calib_l2_gather(const double *table, const int32_t *idx, int64_t n, double *out, int64_t out_len,
                               vjp_stream_t stream);
vjp_status vjp_calib_l2_red(double *table, const int32_t *idx, int64_t n, vjp_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* VJP_B200_H */
