/* =====================================================================================
 *  hodlr2d.h — C ABI of the B200-native HODLR2D fast matrix-vector product.
 *
 *  Method: Kandappan, Gujjula, Ambikasaran, "HODLR2D: A new class of hierarchical
 *  matrices", arXiv 2204.05536.  Citations "P:L" are PAPER.md line numbers.
 *
 *  Problem statement followed by the two main calls (BASELINE.json north_star):
 *    build : given N points, a kernel, N_max and an ACA tolerance epsilon, build the
 *            HODLR2D operator — balanced quadtree, interaction lists I_C and edge sharers
 *            E_C, dense leaf near field, ACA low-rank U V^T for every I_C member
 *            (Alg. 1 "InitializeHODLR2D").
 *    matvec: b = K psi (Alg. 2 "MatVec").
 *  The operator is A = shift*I + scale*K with K_ij = K(|p_i - p_j|), K(0) := K0
 *  (log: 0; IMQ: 1; 1/r: 0, Eq. eq:1byr P:951-958).  See DESIGN.md for every
 *  reading of a point where the paper is silent (R1..R19).
 *
 *  Conventions shared by all calls:
 *   - fp64 only.  Points are interleaved (x, y) pairs, N x 2, in the caller's ORIGINAL
 *     order.  "TREE order" is the Morton order of the quadtree (R4).
 *   - Pointers may be host or device (CUDA) memory; the library detects which with
 *     cudaPointerGetAttributes.  Device pointers must be on the handle's device.
 *   - All device work is ordered on the stream given in the options (default: the
 *     legacy default stream).  With device x/y, matvec is asynchronous w.r.t. the host;
 *     with host x/y it returns after y has been written.
 *   - The handle owns every device allocation it makes; the caller owns points, x, y.
 *   - Return codes: 0 = OK, > 0 = warning, < 0 = error.  The thread-local message of
 *     the last error is returned by hodlr2d_last_error().  A failed build returns no
 *     handle; a handle stays valid after a failed matvec.
 *   - Not thread-safe per handle; distinct handles may be used concurrently.
 * ===================================================================================== */
#ifndef HODLR2D_H
#define HODLR2D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hodlr2d_s* hodlr2d_t; /* opaque handle */

enum {
  H2D_OK = 0,
  H2D_WTRUNC = 1,        /* warning: some ACA block hit max_rank (see info.truncated)      */
  H2D_WNOCONV = 2,       /* warning: hodlr2d_gmres stopped at max_iter above the tolerance  */
  H2D_EINVAL = -1,       /* bad argument: n < 1, leaf_size < 1, tol not in (0,1), NaN/Inf  */
  H2D_EOUTOFBOX = -2,    /* a point lies outside the explicit root box (message: index)    */
  H2D_ECOINCIDENT = -3,  /* reserved (coincident points are legal: K(r=0) := K0, R8)      */
  H2D_ENOMEM = -4,       /* device or host allocation failed                               */
  H2D_ECUDA = -5,        /* CUDA runtime / kernel error                                    */
  H2D_ENCCL = -6,        /* multi-GPU communication error                                  */
  H2D_EFACTORS = -7      /* factor file unreadable or inconsistent with the handle         */
};

enum {
  H2D_KERNEL_LOG = 0,           /* K(r) = log r, K(0) = 0          */
  H2D_KERNEL_IMQ = 1,           /* K(r) = 1/sqrt(1 + (r/c)^2), K(0)=1 (BASELINE configs 2,5) */
  H2D_KERNEL_ONE_OVER_R = 2,    /* K(r) = 1/r, K(0) = 0             (Eq. eq:1byr)  */
  H2D_KERNEL_RBF_PHI1 = 3,      /* phi_1(r) = log r / log a (r >= a), (r log r - 1)/(a log a - 1)
                                   (r < a), K(0) = 0; a = options.c   (Kernel 1) */
  H2D_KERNEL_RBF_PHI2 = 4,      /* phi_2(r) = a / r (r >= a), r / a (r < a), K(0) = 0; a = c
                                                                      (Kernel 2) */
  H2D_KERNEL_TEST_LOWRANK = 100 /* test-only: K(p,q) = sum_{s<test_rank} phi_s(p) phi_s(q),
                                   phi_s(p) = cos((s+1) p.x + 0.5 s p.y) (exact rank)     */
};

/* Orderings of x and y in hodlr2d_matvec_ex:
 *   ORIGINAL : x, y full length N in the caller's point order (single-rank handles);
 *   TREE     : x full length N in TREE order; y = rows [row_begin, row_end) in TREE order;
 *   GATHERED : x = world slots of info.gather_stride values, slot r holding rank r's TREE
 *              rows [row_begin_r, row_end_r) followed by padding — exactly the output of one
 *              equal-count all-gather (ncclAllGather / all_gather_into_tensor) of every
 *              rank's padded slice; y as for TREE. */
enum { H2D_ORDER_ORIGINAL = 0, H2D_ORDER_TREE = 1, H2D_ORDER_GATHERED = 2, H2D_ORDER_LOCAL = 3 };
/*   LOCAL    : x = this rank's TREE rows [row_begin, row_end) only; the library all-gathers
 *              the slices of every rank itself (S11; the paper's distributed
 *              matvec, §6) through the handle's communicator (options.nccl_id or
 *              options.allgather) and overlaps it with the stage-A items whose column box is
 *              local; y as for TREE.  Every rank of the world must call it (collective). */

/* Bytes of the NCCL unique id carried by options.nccl_id (ncclUniqueId). */
#define H2D_COMM_ID_BYTES 128

/* Host all-gather callback (options.allgather): gather bytes_per_rank bytes of `send` from
 * every rank of the world into `recv` (world * bytes_per_rank bytes, rank order), both host
 * memory owned by the library; return 0 on success.  For worlds without NCCL between the
 * ranks (e.g. several ranks sharing one GPU in tests); the library calls it from inside
 * hodlr2d_matvec_ex(..., H2D_ORDER_LOCAL) on the calling thread. */
typedef int (*hodlr2d_allgather_fn)(const void* send, void* recv, size_t bytes_per_rank, void* ctx);

/* Options of hodlr2d_build_ex.  Always start from hodlr2d_default_options(). */
typedef struct {
  double c;               /* IMQ shape c > 0; RBF phi_1/phi_2 parameter a > 0  (default 1)  */
  double scale;           /* A = shift*I + scale*K                             (default 1)  */
  double shift;           /*                                                   (default 0)  */
  double box_lo[2];       /* root square lower-left corner                                  */
  double box_side;        /* root square side; <= 0 -> bounding square of the points (R2)   */
  int depth;              /* kappa >= 0; -1 -> R1 depth rule (nominal leaf size); -2 -> the
                             paper's rule (Alg. 1 l.3): smallest kappa with no leaf
                             holding more than leaf_size points (R22); -3 -> the adaptive
                             (non-balanced) quadtree of P:914 (R24): a box is split iff it
                             holds more than leaf_size points; single-rank handles, directed
                             apply (multi-RHS calls loop over vectors)     (default -1) */
  int max_rank;           /* ACA rank cap per block; hitting it sets H2D_WTRUNC (def. 128)  */
  int aca_consecutive;    /* tolerance hits in a row that stop ACA (R7)        (default 3)  */
  int aca_trim;           /* streak terms dropped on a tolerance stop (R7)     (default 3)  */
  int test_rank;          /* H2D_KERNEL_TEST_LOWRANK only                      (default 1)  */
  void* stream;           /* cudaStream_t for all work                         (default 0)  */
  int world;              /* Morton-range partition: number of ranks           (default 1)  */
  int rank;               /* this rank, 0 <= rank < world                      (default 0)  */
  int64_t row_begin;      /* explicit served TREE-order range [row_begin, row_end) snapped  */
  int64_t row_end;        /*   to leaf boundaries; row_end <= 0 -> from world/rank (def 0)  */
  size_t aca_scratch_bytes; /* ACA scratch budget; 0 -> 40 % of free device memory         */
  int timing;             /* 1 -> record per-stage CUDA events in every matvec (default 0)  */
  int skip_aca;           /* 1 -> build tree + lists only (factors via load_factors)        */
  int symmetric;          /* 1 -> one ACA per unordered pair {X, Y}, X < Y in Morton order;
                             block (Y, X) := V U^T (the paper's symmetric setting, P:61;
                             halves the ACA work, exactly symmetric operator, R23)  (def 0) */
  const double* leaf_weights; /* world > 1: host array of 4^kappa per-leaf loads (the same on
                             every rank) replacing the geometric weight of the Morton-range
                             partition — e.g. the sum over ranks of hodlr2d_leaf_costs from a
                             first build; kappa must match.  Not copied.     (default NULL) */
  const unsigned char* nccl_id; /* H2D_COMM_ID_BYTES-byte NCCL unique id (rank 0 calls
                             hodlr2d_comm_unique_id, the caller broadcasts it, e.g. with
                             torch.distributed): the handle creates and owns an NCCL
                             communicator of `world` ranks (ncclCommInitRank, collective over
                             the ranks) and its gather buffer (ncclMemAlloc + ncclCommRegister);
                             enables H2D_ORDER_LOCAL.  Copied.               (default NULL) */
  hodlr2d_allgather_fn allgather; /* host-staged alternative to nccl_id (used when nccl_id is
                             NULL); enables H2D_ORDER_LOCAL                  (default NULL) */
  void* allgather_ctx;    /* passed to allgather                             (default NULL) */
} hodlr2d_options;

#define H2D_MAX_LEVELS 16
#define H2D_NUM_STAGES 6 /* 0 input permute / unpad, 1 stage A (t = V^T x, incl. the
                            multi-chunk t reduction), 2 stage B (yfar = U t), 3 wait for
                            the near-field P2P after stage B, 4 combine (y = yfar + scale
                            K_near x + shift x, output permutation), 5 near-field P2P (runs
                            on a low-priority stream concurrently with stages 1-2)     */

typedef struct {
  int64_t n;                 /* N                                                     */
  int kappa;                 /* tree depth                                            */
  int world, rank;
  int64_t row_begin, row_end;/* TREE-order rows this handle serves                    */
  int64_t leaf_begin, leaf_end;
  double box_lo[2], box_side;
  int64_t blocks_per_level[H2D_MAX_LEVELS + 1]; /* directed blocks (all, l = 1..kappa)   */
  int64_t blocks_built;      /* blocks this handle stores                             */
  int rank_max;              /* r_m                                           */
  int64_t rank_hist[129];    /* blocks with rank r (r >= 128 -> bin 128)               */
  int64_t u_values, v_values;/* stored fp64 factor values (U and V panels)            */
  int64_t near_pairs;        /* sum over served leaves of |X| * |{X} u E_X|           */
  double compression_ratio;  /* (factor values + near pairs) / N^2  (CR)        */
  int64_t truncated;         /* blocks that hit max_rank                              */
  double tree_seconds, aca_seconds, pack_seconds, build_seconds;
  int64_t matvec_bytes;      /* algorithmic HBM bytes of one matvec */
  int64_t stageA_bytes, stageB_bytes;
  double p2p_pairs;          /* near-field pair evaluations per matvec                */
  int64_t device_bytes;      /* device memory held by the handle                      */
  int64_t gather_stride;     /* max rows over ranks (slot size of H2D_ORDER_GATHERED) */
  int64_t p2p_bytes;         /* algorithmic bytes of the near-field P2P kernel        */
  int symmetric_apply;       /* 1 -> matvecs run the symmetric three-pass apply (R23;
                                every symmetric build unless H2D_SYMAPPLY=0, a rank of a
                                partition too): stage slot 1 = A' + B', slot 2 = C';
                                stageA_bytes / stageB_bytes then count those passes    */
  int p2p_launches;          /* near-field kernels per matvec: warp-per-leaf (one per rows-
                                per-lane class 1..3, leaves <= 96 points), CTA fast path,
                                generic (1..5)                                         */
  int64_t p2p_leaves[3];     /* leaves on the warp / fast / generic P2P paths          */
  int apply_launches;        /* low-rank apply kernels per matvec: stage A / B rings and
                                their small-item (warp-per-item) kernels, B' (symmetric) */
  int64_t small_items[2];    /* stage A boxes / stage B leaves on the small-item kernels */
  int comm_kind;             /* 0 none, 1 NCCL communicator, 2 host all-gather callback  */
  int adaptive;              /* 1: adaptive quadtree (depth = -3, R24)          */
  int pair_apply;            /* 1: matvecs run the pair-local symmetric apply (symmetric
                                single-rank handles: each factor read once)
                                and stageA_bytes counts its pass                         */
  int64_t n_leaves;          /* leaves (adaptive: hodlr2d_copy_leaves; else 4^kappa)      */
  int64_t local_items[2];    /* H2D_ORDER_LOCAL: stage-A items (ring, small) whose column box
                                is local, run while the x all-gather is in flight        */
  int64_t stored_near_values;/* fp64 values of the stored near-field blocks that 16-vector
                                multi-RHS chunks read (Alg. 1 l.5; built on the
                                first such call, 0 before it or when it did not fit)     */
  int p2p_log_table;         /* log table of the near field (the warp-per-leaf kernel; on
                                adaptive handles the list kernel, log and phi_1): 0 the
                                512-bin table, 1 the replicated 64-bin table (picked at
                                build by timing both), -1 none (other
                                kernels, or the subnormal-safe log)                      */
} hodlr2d_info;

/* Fill *opts with the defaults listed above. */
void hodlr2d_default_options(hodlr2d_options* opts);

/* Build with default options (c = 1, scale = 1, shift = 0, bounding-square root box,
 * R1 depth rule).  points: N x 2 fp64 (host or device), copied; n >= 1; leaf_size >= 1
 * (N_max of Alg. 1); aca_tol in (0, 1).  *out receives the handle on success (return
 * 0 or H2D_WTRUNC), is set to NULL on error. */
int hodlr2d_build(const double* points, int64_t n, int kernel_id, int leaf_size, double aca_tol,
                  hodlr2d_t* out);

/* Same with explicit options (root box, kernel parameters, partition, stream ...). */
int hodlr2d_build_ex(const double* points, int64_t n, int kernel_id, int leaf_size, double aca_tol,
                     const hodlr2d_options* opts, hodlr2d_t* out);

/* y = A x, both length N in ORIGINAL order (single-rank handles).  y is overwritten. */
int hodlr2d_matvec(hodlr2d_t h, const double* x, double* y);

/* y = A x with an explicit ordering.  order = H2D_ORDER_TREE: x is the full length-N
 * vector in TREE order and y receives rows [row_begin, row_end) in TREE order
 * (length row_end - row_begin).  order = H2D_ORDER_GATHERED: x is the padded
 * all-gather buffer (world * info.gather_stride values, see the enum above); the library
 * unpads it into its TREE-order x inside the matvec.  order = H2D_ORDER_ORIGINAL: as
 * hodlr2d_matvec (single-rank handles only). */
int hodlr2d_matvec_ex(hodlr2d_t h, const double* x, double* y, int order);

/* Stream-ordered y = A x for a sequence of matvecs on host buffers (the same operation as
 * hodlr2d_matvec_ex, Alg. 2 of the paper): enqueues the host -> device copy of x,
 * the matvec and the device -> host copy of y, and RETURNS BEFORE THEY RUN.  x and y must be
 * pinned host memory (cudaMallocHost / cudaHostRegister / torch pin_memory) or device
 * memory; order = H2D_ORDER_ORIGINAL, TREE or GATHERED with the lengths of hodlr2d_matvec_ex.
 * The copies run on two library-owned streams (one per copy engine) and the library keeps two
 * device staging slots, so call k + 1's upload and call k - 1's download overlap call k's
 * kernels.  Ownership: the caller must not modify x or read y until hodlr2d_wait(h) returns
 * (which waits for every call enqueued so far); the library owns the staging buffers.
 * Results are bitwise those of hodlr2d_matvec_ex.  Errors: H2D_EINVAL for pageable host
 * buffers, a null pointer, LOCAL order or a bad order/handle combination (nothing is
 * enqueued); asynchronous CUDA errors surface from hodlr2d_wait as H2D_ECUDA. */
int hodlr2d_matvec_async(hodlr2d_t h, const double* x, double* y, int order);

/* Block until every hodlr2d_matvec_async call on h has completed (its y written). */
int hodlr2d_wait(hodlr2d_t h);

/* Y = A X for nrhs vectors at once (NEXT N2; the paper applies its matvec to ten input
 * vectors).  Vector k is X + k * len_x and Y + k * len_y; order =
 * H2D_ORDER_ORIGINAL (single-rank handles, len_x = len_y = N), H2D_ORDER_TREE (x in TREE
 * order, len_x = N, y = the served rows, len_y = row_end - row_begin) or
 * H2D_ORDER_GATHERED (x = one padded all-gather buffer per vector, len_x = world *
 * info.gather_stride; y as for TREE).  The factor panels are streamed once per chunk of up
 * to 16 vectors (chunks of 16, 8, 4, 2; a last single vector takes the hodlr2d_matvec
 * path; symmetric-apply handles: chunks of 8, one vector at a time on a rank of a
 * partition), so throughput in matvecs/s grows with nrhs
 * until the FP64 pipes, not HBM, bound it.  Host or device pointers; Y is overwritten.
 * Results equal nrhs separate hodlr2d_matvec_ex calls up to rounding (different
 * summation order). */
int hodlr2d_matvec_multi(hodlr2d_t h, const double* X, double* Y, int nrhs, int order);

/* Solve A x = b with restarted GMRES(restart) accelerated by the HODLR2D matvec — the
 * iterative solver of the paper's applications (§5: ACA tolerance 1e-12 and GMRES residual
 * 1e-10; RBF interpolation with phi_1 / phi_2; R20).
 * b, x: length N in ORIGINAL order, host or device pointers; x0 = 0 and x is overwritten.
 * Arnoldi with classical Gram-Schmidt + one reorthogonalisation, Givens rotations; stops
 * when the estimated relative residual ||b - A x|| / ||b|| < tol (checked against the true
 * residual at every restart) or after max_iter Arnoldi steps.  *iters (may be NULL)
 * receives the Arnoldi steps (= matvecs excluding restarts), *rel_residual (may be NULL)
 * the TRUE relative residual of the returned x.  Single-rank handles only.  Returns
 * H2D_OK, H2D_WNOCONV if tol was not reached, or an error. */
int hodlr2d_gmres(hodlr2d_t h, const double* b, double* x, double tol, int restart, int max_iter,
                  int* iters, double* rel_residual);

/* Statistics of the built operator (host struct). */
int hodlr2d_get_info(hodlr2d_t h, hodlr2d_info* info);

/* Copy the tree to host arrays: perm[N] (TREE position -> ORIGINAL index) and
 * leaf_start[4^kappa + 1].  Either pointer may be NULL. */
int hodlr2d_copy_tree(hodlr2d_t h, int32_t* perm, int32_t* leaf_start);

/* Copy the CSR interaction list of level 1 <= level <= kappa to host arrays:
 * off[4^level + 1], col[off[4^level]] (partner Morton index, ascending).
 * level = 0 copies the leaf near field {X} u E_X (off[4^kappa + 1]). */
int hodlr2d_copy_lists(hodlr2d_t h, int level, int32_t* off, int32_t* col);

/* Leaves of the tree in Morton order: level[] and box[] (box index at that level) of each;
 * returns their count (either array may be NULL).  Balanced trees: the 4^kappa boxes of level
 * kappa; adaptive trees (depth = -3, R24): the unsplit boxes at their own levels.  -1 for a
 * NULL handle. */
int64_t hodlr2d_copy_leaves(hodlr2d_t h, int32_t* level, int32_t* box);

/* Number of directed blocks of a level (CSR length); -1 if level is out of range. */
int64_t hodlr2d_num_blocks(hodlr2d_t h, int level);

/* Ranks of the blocks of one level in CSR order (host array); -1 = not stored by this rank. */
int hodlr2d_copy_ranks(hodlr2d_t h, int level, int32_t* ranks);

/* Copy the factors of block `e` (CSR order) of `level` to host: U (m x r) and V (n x r),
 * column-major.  Pass NULL arrays to query m, n, r only. */
int hodlr2d_copy_block(hodlr2d_t h, int level, int64_t e, int* m, int* n, int* r, double* U,
                       double* V);

/* Replace the factors by those of an oracle interchange file (R11); the file's
 * N, kappa and perm must match the handle.  Used for the oracle-factor parity test. */
int hodlr2d_load_factors(hodlr2d_t h, const char* path);

/* Write the handle's factors in the same interchange format (single-rank handles). */
int hodlr2d_save_factors(hodlr2d_t h, const char* path);

/* Accumulated device time (ms) per stage over the matvecs run since the last reset,
 * measured with CUDA events on the handle's stream (options.timing = 1).  ms[] has
 * H2D_NUM_STAGES entries; *count receives the number of matvecs.  Synchronises. */
int hodlr2d_stage_times(hodlr2d_t h, double* ms, int64_t* count, int reset);

/* Enable / disable stage timing after the build. */
int hodlr2d_set_timing(hodlr2d_t h, int on);

/* Measured load of the handle's served leaves, for a load-balanced re-partition: costs
 * (host, 4^kappa entries) receives for every served leaf L the algorithmic bytes of one
 * matvec attributable to it — 8 |L| (sum over L's ancestors X of the U columns of X plus
 * the V columns of X's column box) + 24 |L| — and 0 for leaves the handle does not serve.
 * Summed over the ranks of a world it is the leaf_weights option of a rebuild.  Host
 * computation from the packed layout (no device work). */
int hodlr2d_leaf_costs(hodlr2d_t h, double* costs);

/* Host-only helper (no device work; callable without a GPU): the Morton-range partition
 * every rank of a world uses.  leaf_start: the tree's 4^kappa + 1 leaf
 * offsets (see hodlr2d_copy_tree); n = leaf_start[4^kappa].  Rank r serves leaves
 * [*leaf_begin, *leaf_end): contiguous Morton ranges cut at the quantiles r / world of the
 * per-leaf load w(L) = |L| (1 + sum over L's ancestors X of |I_X|) — rows times the blocks
 * they meet, the geometric part of Eq. eq:par's per-node load — each cut
 * snapped to a coarse box boundary when that shifts at most 3 % (level 1) / 4 % (level 2) /
 * 4x less per finer level of a rank's share (a cut inside a box makes both ranks stream
 * the V panels of all its partners).  leaf_start must hold 4^kappa + 1 entries; kappa <= 15.
 * Errors: H2D_EINVAL (bad arguments), H2D_ENOMEM (host allocation). */
int hodlr2d_partition(const int32_t* leaf_start, int kappa, int world, int rank,
                      int64_t* leaf_begin, int64_t* leaf_end);

/* Diagnostics switches of one handle's matvec (none changes results beyond
 * rounding order, except "dual_norow", which skips the symmetric B' row dots and gives WRONG
 * results, for timing only): "p2p_serial" (the near field alone, before stage A),
 * "p2p_onestream" (every near-field class on one stream), "dual_norow", "copy_stream" (0:
 * host copies on the work stream), "pair_apply" (symmetric handles: 1 the pair-local apply,
 * 0 the three-pass apply), "multi_stored_near" (16-vector multi-RHS chunks: 1 (default) the
 * stored dense near-field blocks of Alg. 1 l.5, built on the first such call when they
 * fit in half the free device memory; 0 the on-the-fly near field), "multi_log_table"
 * (multi-RHS on-the-fly log near field: 1 (default) the replicated 64-bin log table, 0 the
 * 512-bin one), "p2p_place" (directed matvecs: 0 (default) the near field beside stage A,
 * 1 beside stage B, -1 timed on matvec calls 1-4; results bit-identical; H2D_EINVAL outside
 * -1..1).  Defaults come from the H2D_* environment variables at build time.  H2D_EINVAL for
 * an unknown name. */
int hodlr2d_set_diag(hodlr2d_t h, const char* name, int value);

/* Write a fresh NCCL unique id (H2D_COMM_ID_BYTES bytes) to id[] for options.nccl_id
 * (called on one rank, then broadcast).  H2D_ENCCL if NCCL cannot be loaded. */
int hodlr2d_comm_unique_id(unsigned char* id);

/* Release every resource of the handle.  NULL is accepted. */
int hodlr2d_destroy(hodlr2d_t h);

/* Message of the last error on this thread ("" if none). */
const char* hodlr2d_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HODLR2D_H */
