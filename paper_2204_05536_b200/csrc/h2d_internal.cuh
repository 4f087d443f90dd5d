// Internal declarations of the B200 HODLR2D library (not part of the C ABI).
// Product code only: nothing here is shared with oracle/ (DESIGN.md §Independence).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/hodlr2d.h"

namespace h2d {

// ------------------------------------------------------------------ errors
struct Error {
  int code;
  std::string msg;
};
void set_error(int code, const std::string& msg);
#define H2D_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      throw ::h2d::Error{_e == cudaErrorMemoryAllocation ? H2D_ENOMEM : H2D_ECUDA,        \
                         std::string(#call) + ": " + cudaGetErrorString(_e) + " at " +    \
                             __FILE__ + ":" + std::to_string(__LINE__)};                  \
  } while (0)
#define H2D_LAUNCH_CHECK() H2D_CUDA(cudaGetLastError())

// ------------------------------------------------------------------ kernel entries
struct KernelParams {
  int id;          // H2D_KERNEL_*
  double inv_c2;   // 1 / c^2 (IMQ)
  double a, a2;    // RBF parameter a and a^2 (phi_1, phi_2)
  double inv_log_a;      // 1 / log a                 (phi_1, r >= a)
  double inv_phi1_den;   // 1 / (a log a - 1)         (phi_1, r < a)
  double scale;    // A = shift I + scale K
  double shift;
  int test_rank;
};

// Internal kernel id of the near-field kernels: the log kernel with subnormal-safe table
// logarithms (handles whose near field has a pair of distinct points with subnormal r^2).
constexpr int kLogSafe = 5;
// ... and the log kernel without the K(r = 0) select in the warp-per-leaf near field (handles
// whose near field has no two distinct points at distance 0 and no subnormal r^2): the self
// block's diagonal term is taken out once per row instead of a select per evaluation.
constexpr int kLogNoSel = 6;
// ... and the same with the replicated 64-bin log table (pipe.cuh hlog_r2<false, true>): no
// shared-memory bank conflicts on the table lookups, two more DFMAs per evaluation; the build
// times both on the handle's own near field and keeps the faster (apply.cu pick_log_table).
constexpr int kLogNoSelRepl = 7;
// ... and the replicated table in the adaptive list near field (p2p_list_kernel): the log
// kernel (with the K(0) select) and the RBF phi_1 kernel (apply.cu pick_list_table).
constexpr int kLogRepl = 8, kPhi1Repl = 9;

// K(p, q) specialised at compile time (hot P2P loop: no per-pair dispatch).
template <int KID>
__device__ __forceinline__ double kernel_eval_t(const KernelParams& k, double px, double py,
                                                double qx, double qy) {
  const double dx = px - qx, dy = py - qy;
  const double r2 = fma(dx, dx, dy * dy);
  if (KID == H2D_KERNEL_LOG || KID == kLogSafe || KID == kLogNoSel || KID == kLogNoSelRepl || KID == kLogRepl) {
    return r2 > 0.0 ? 0.5 * log(r2) : 0.0;
  } else if (KID == H2D_KERNEL_IMQ) {
    return rsqrt(fma(r2, k.inv_c2, 1.0));
  } else if (KID == H2D_KERNEL_ONE_OVER_R) {
    return r2 > 0.0 ? rsqrt(r2) : 0.0;
  } else if (KID == H2D_KERNEL_RBF_PHI1 || KID == kPhi1Repl) {
    if (r2 == 0.0) return 0.0;
    if (r2 >= k.a2) return 0.5 * log(r2) * k.inv_log_a;
    const double r = sqrt(r2);
    return fma(r, log(r), -1.0) * k.inv_phi1_den;
  } else if (KID == H2D_KERNEL_RBF_PHI2) {
    if (r2 >= k.a2) return k.a * rsqrt(r2);
    return sqrt(r2) / k.a;
  } else {
    double acc = 0.0;
    for (int s = 0; s < k.test_rank; ++s)
      acc = fma(cos((s + 1) * px + 0.5 * s * py), cos((s + 1) * qx + 0.5 * s * qy), acc);
    return acc;
  }
}

// K(p, q) for r^2 = |p - q|^2; K(r = 0) := K0 (R8) by distance, not by index.
__device__ __forceinline__ double kernel_eval(const KernelParams& k, double px, double py,
                                              double qx, double qy) {
  double dx = px - qx, dy = py - qy;
  double r2 = fma(dx, dx, dy * dy);
  if (k.id == H2D_KERNEL_LOG) {
    return r2 > 0.0 ? 0.5 * log(r2) : 0.0;
  } else if (k.id == H2D_KERNEL_IMQ) {
    return rsqrt(fma(r2, k.inv_c2, 1.0));
  } else if (k.id == H2D_KERNEL_ONE_OVER_R) {
    return r2 > 0.0 ? rsqrt(r2) : 0.0;
  } else if (k.id == H2D_KERNEL_RBF_PHI1) {
    return kernel_eval_t<H2D_KERNEL_RBF_PHI1>(k, px, py, qx, qy);
  } else if (k.id == H2D_KERNEL_RBF_PHI2) {
    return kernel_eval_t<H2D_KERNEL_RBF_PHI2>(k, px, py, qx, qy);
  } else {
    double acc = 0.0;
    for (int s = 0; s < k.test_rank; ++s)
      acc = fma(cos((s + 1) * px + 0.5 * s * py), cos((s + 1) * qx + 0.5 * s * qy), acc);
    return acc;
  }
}

// ------------------------------------------------------------------ operator storage
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Level {
  int l = 0;
  int64_t nbox = 0;          // 4^l
  int64_t nblocks = 0;       // directed blocks (CSR length)
  // lists (device + host copy)
  int32_t* d_off = nullptr;  // [nbox + 1]
  int32_t* d_col = nullptr;  // [nblocks]
  std::vector<int32_t> off, col;
  std::vector<int32_t> trans;  // block id of (Y, X) for block (X, Y)
  // per block (host): rank, built flag, panel columns
  std::vector<int32_t> rank;   // -1 = not built on this rank
  std::vector<uint8_t> truncated;
  std::vector<int32_t> ucol;   // first column of the block among the U columns of its row box
  std::vector<int32_t> vcol;   // first column inside the V panel of the column box
  // U leaf panels (device): for every served leaf L with level-l ancestor X, the rows of L
  // of all U columns of X ([U_b1 | U_b2 | ...], blocks (X, Y), Y in I_X ascending):
  // column-major mLp x R_X at U + uoff[L - leaf_begin], mLp = |L| rounded up to even, so a
  // leaf's level-l factors are one contiguous, 16-byte aligned range (bulk-TMA source).
  // V panel of column box Y: row-major n_Y x RVp_Y at V + vpan_off[Y], RVp_Y = RV_Y
  // rounded up to even (every row chunk is a 16-byte aligned range).
  double* U = nullptr;
  double* V = nullptr;
  int64_t u_values = 0, v_values = 0;       // stored factor values (without padding)
  int64_t u_alloc = 0, v_alloc = 0;         // allocated doubles (with padding)
  std::vector<int64_t> uoff;                // per served leaf
  std::vector<int64_t> vpan_off;            // per box
  std::vector<int32_t> ucolbase;            // per box + 1 (prefix of R_X)
  std::vector<int32_t> vR;                  // per box RV_Y
  std::vector<int64_t> t_off;               // per box: first vdst entry of column box Y
  int32_t* d_ucolbase = nullptr;            // [nbox + 1]
  int64_t* d_uoff = nullptr;                // [served leaves]
  int64_t tu_base = 0;                      // first t entry of the level (U-column order)
  // symmetric apply (Handle::symapply): the U leaf / V box panels above then hold the
  // second-side blocks (Y, X), Y > X (U leaf panels, = V of the pair) and the first-side
  // blocks (Z, Y), Z < Y (V box panels); the first-side U factors (X, Y), X < Y, are kept
  // as row-major box panels Ub (m_X x ubRp_X) for stage B' of the symmetric matvec.
  double* Ub = nullptr;
  int64_t ub_values = 0, ub_alloc = 0;
  std::vector<int64_t> ub_off;              // per box
  std::vector<int32_t> ubR;                 // per box: first-side columns R^F_X
  std::vector<int32_t> ubcol;               // per block (first side): column in the Ub panel of X
  std::vector<int32_t> t1base;              // per box + 1: prefix of R^F (t1 layout)
  int64_t t1_base = 0;                      // first t1 entry of the level
  // pair apply (Handle::pairapply): per pair {X, Y}, X < Y, rank r > 0, V (n_Y x Rp) then
  // U (m_X x Rp), row-major, Rp = r rounded up to even (zero pad column), in Pr
  struct PairDesc {
    int64_t v_off, u_off;
    int32_t yv, yu, nv, nu, R, Rp;
  };
  double* Pr = nullptr;
  int64_t pr_values = 0, pr_alloc = 0;
  std::vector<PairDesc> pairs;
};

// Stage-A work item: one row chunk of one V panel.  Outputs go to t (U-panel order)
// through vdst[out + q] when out >= 0, or to the partial buffer at -out-1 + q.
struct AItem {
  int64_t v_off;   // element offset of the chunk's first row inside the level V array
  int64_t x_off;   // TREE index of the chunk's first row
  int32_t nrows;
  int32_t R;       // panel width RV_Y
  int32_t out;
  int32_t level;
  int32_t ritem;   // >= 0: multi-chunk box (RItem index); the last chunk CTA reduces
  int32_t Rp;      // row stride of the panel (R rounded up to even)
  int64_t t1_off;  // symmetric stage B': first t1 entry of the item's row box (else 0)
};
// Stage-B work item: rows [r0, r0 + rows) (rows <= 224) of a served leaf of mL points whose
// first output row is yrow (index into the served rows); its per-level metadata is
// BLevel[item * kappa + l - 1].
struct BItem {
  int32_t r0;
  int32_t rows;
  int32_t mL;
  int32_t yrow;
};
struct BLevel {
  int64_t uoff;    // leaf-panel offset inside the level's U array
  int32_t tcol;    // first t entry of the level-l ancestor box (U-column order)
  int32_t R;       // U columns of that box
};
// Reduction of multi-chunk partials: t[vdst[vpos + q]] = sum_c part[p_off + c*R + q]
struct RItem {
  int32_t vpos;
  int32_t p_off;
  int32_t R;
  int32_t nchunks;
};

// Run f() once per (call site, current device): kernel function attributes (dynamic smem
// size, carve-out) belong to a device's context, so a process driving several GPUs must set
// them on each.  `seen` is the call site's device bitmask; the mutex also orders a second
// thread after the first one's attribute calls.
template <typename F>
inline void once_per_device(uint64_t& seen, F&& f) {
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> lock(mu);
  if (seen & bit) return;
  f();
  seen |= bit;
}

struct LevelPtrs {
  const double* U[H2D_MAX_LEVELS + 1];
  const double* V[H2D_MAX_LEVELS + 1];
  const int32_t* ucolbase[H2D_MAX_LEVELS + 1];
  const int64_t* uoff[H2D_MAX_LEVELS + 1];  // U leaf-panel offsets (served leaves)
  const double* tu[H2D_MAX_LEVELS + 1];   // t of the level in U-column order
  const double* Ub[H2D_MAX_LEVELS + 1];   // symmetric apply: first-side U box panels
};

struct Comm;   // comm.cu: the handle's communicator (S11)

struct Handle {
  int device = 0;
  cudaStream_t stream = 0;
  hodlr2d_options opts{};
  KernelParams kp{};
  int kernel_id = 0;
  int leaf_size = 0;
  double tol = 0;
  int64_t n = 0;
  int kappa = 0;
  double lo[2] = {0, 0}, side = 1;
  int64_t row_begin = 0, row_end = 0;     // served TREE rows
  int64_t leaf_begin = 0, leaf_end = 0;   // served leaves
  std::vector<int64_t> rank_rows;         // [world + 1] first TREE row of every rank
  int64_t* d_rank_rows = nullptr;
  int64_t gather_stride = 0;              // max rows over ranks (padded all-gather slot)
  // tree (device)
  double* d_px = nullptr;
  double* d_py = nullptr;
  int32_t* d_perm = nullptr;
  int32_t* d_leaf_start = nullptr;
  std::vector<int32_t> leaf_start;        // host copy
  // Adaptive quadtree (options.depth = -3, R24): a box is subdivided iff it holds
  // more than N_max points.  The "leaves" every per-leaf structure below iterates (U leaf
  // panels, stage-B items, the near field) are then the adaptive leaves, at various levels:
  // lf_code = index of the leaf's first level-kappa descendant (its level-l ancestor is
  // lf_code >> 2 (kappa - l)), lf_start = its TREE-order rows.  Balanced handles: the 4^kappa
  // level-kappa boxes (lf_code = identity, lf_start = leaf_start).
  bool adaptive = false;
  std::vector<std::vector<uint8_t>> ad_sub;   // [level][box]: subdivided (exists iff parent subdivided)
  std::vector<int64_t> lf_code;
  std::vector<int32_t> lf_start, lf_level;
  // the adaptive near field, per served leaf: column ranges (TREE begin, count) of every dense
  // block whose row box contains the leaf (R24); CSR over leaves
  std::vector<int64_t> ad_nf_off;
  std::vector<int64_t> ad_nf_rng;   // pairs (begin, count)
  int64_t* d_p2p_list = nullptr;   // items (leaf << 8 | 64-row pass) of the list kernel
  int64_t n_p2p_list = 0;
  int64_t* d_ad_nf_off = nullptr;
  int64_t* d_ad_nf_rng = nullptr;
  int32_t* d_lf_start = nullptr;
  int64_t leaf_code(int64_t lf) const { return adaptive ? lf_code[(size_t)lf] : lf; }
  int64_t leaf_s(int64_t lf) const { return adaptive ? lf_start[(size_t)lf] : leaf_start[(size_t)lf]; }
  int64_t leaf_e(int64_t lf) const { return adaptive ? lf_start[(size_t)lf + 1] : leaf_start[(size_t)lf + 1]; }
  int leaf_level(int64_t lf) const { return adaptive ? lf_level[(size_t)lf] : kappa; }
  bool box_exists(int l, int64_t b) const { return !adaptive || l == 0 || ad_sub[(size_t)l - 1][(size_t)(b >> 2)]; }
  // near field (device + host)
  int32_t* d_nf_off = nullptr;
  int32_t* d_nf_col = nullptr;
  std::vector<int32_t> nf_off, nf_col;
  // levels 1..kappa
  std::vector<Level> levels;
  // stage A / reduce schedule
  AItem* d_aitems = nullptr;
  int64_t n_aitems = 0;
  RItem* d_ritems = nullptr;
  int64_t n_ritems = 0;
  int32_t* d_rcount = nullptr;            // per RItem: chunk CTAs finished (self-resetting)
  double* d_t = nullptr;                  // all t values, U-panel column order
  int32_t* d_vdst = nullptr;              // V-panel column (column-box order) -> t index
  int64_t t_len = 0;
  double* d_tpart = nullptr;              // multi-chunk partials
  int64_t tpart_len = 0;
  LevelPtrs lp{};
  int rmax_panel = 1;                     // widest per-leaf t gather (smem of stage B)
  int max_ritem_R = 1;
  BItem* d_bitems = nullptr;              // stage-B items, largest first
  BLevel* d_blev = nullptr;               // [n_bitems * kappa]
  int64_t n_bitems = 0;
  int32_t* d_counters = nullptr;          // dynamic work counters: stage A, B, P2P fast, B', P2P warp
  int persist_ctas = 0;                   // CTAs of the persistent stage-A/B kernels
  int pipe_ns = 0;                        // their ring depth (template instance)
  int num_sms = 0;
  int32_t* d_p2p_fast = nullptr;          // leaves of the persistent fast P2P kernel
  int32_t* d_p2p_gen = nullptr;           // leaves of the generic P2P kernel
  int64_t n_p2p_fast = 0, n_p2p_gen = 0;
  int64_t n_abig = 0, n_bbig = 0;         // stage A / B items on the ring (the rest: small-item kernels)
  // H2D_ORDER_LOCAL (communicator): the stage-A items whose column box lies in the served
  // rows come first in both the ring and the small-item lists; they run during the gather
  Comm* comm = nullptr;
  int64_t n_abig_loc = 0, n_asmall_loc = 0;
  int32_t* d_p2p_warp = nullptr;          // <= 32-point leaves of the warp-per-leaf P2P kernel
  int64_t n_p2p_warp = 0;
  int64_t n_p2p_warp_rpl[3] = {0, 0, 0};  // warp-kernel leaves with 1 / 2 / 3 rows per lane
  // symmetric apply (symmetric build on a single-rank handle, R23): A' over the
  // first-side V box panels -> t1; B' over the first-side U box panels -> t2 (= t) and the
  // per-level row dots y1 = U t1; C' = stage B over the second-side leaf panels with t2
  bool symapply = false;
  bool small_a_after = false;
  bool p2p_after_b1 = false;    // H2D_P2P_AFTER_B1=1: symmetric near field waits for B' (beside C' only)
  cudaEvent_t ev_b1 = nullptr;   // H2D_SMALL_A_AFTER=1: the small stage-A kernel after the ring
  double* d_t1 = nullptr;                 // [t1_len]
  int64_t t1_len = 0;
  int32_t* d_udst = nullptr;              // U-box column -> t2 index
  AItem* d_b1items = nullptr;             // stage B' items
  int64_t n_b1items = 0;
  int64_t n_b1big = 0;                   // B' ring items (the rest: stageB1_small_kernel)
  RItem* d_b1ritems = nullptr;
  int32_t* d_b1rcount = nullptr;
  double* d_b1tpart = nullptr;
  double* d_y1 = nullptr;                 // [kappa][n] per-level row dots of B'
  // pair-local symmetric apply (pairs.cuh): every factor read once per matvec
  bool pairapply = false;
  bool pair_wanted = false;               // symmetric single-rank handle (H2D_PAIRAPPLY != 0)
  bool pair_failed = false;               // a rank above 127 in the current factors
  void* d_pitems = nullptr;               // PWork[]
  void* d_ppairs = nullptr;               // PPair[]
  int64_t n_pitems = 0;
  double *d_tP1 = nullptr, *d_tP2 = nullptr, *d_ptpart = nullptr;
  int32_t *d_pcount = nullptr, *d_pflags = nullptr;
  int pair_epoch = 0;
  int pair_ctas_per_sm = 2;
  int64_t pair_values = 0;                // factor values the pair kernel streams (U + V)
  double* d_yacc = nullptr;               // [n] TREE-order accumulator of the pair kernel
  // multi-RHS (multi.cu): tiled stage-A schedule and per-chunk buffers (<= 8 vectors)
  bool multi_ready = false;
  AItem* m_aitems = nullptr;
  int64_t m_n_aitems = 0;
  RItem* m_ritems = nullptr;
  int32_t* m_rcount = nullptr;
  double *m_tpart = nullptr, *m_xm = nullptr, *m_t = nullptr;
  int32_t* m_iperm = nullptr;             // inverse of d_perm (ORIGINAL index -> TREE row)
  double *m_yfar = nullptr, *m_ynear = nullptr;
  // 16-vector chunks: stage-A tiles of <= 224 columns (their own schedule)
  AItem* m16_aitems = nullptr;
  int64_t m16_n_aitems = 0;
  RItem* m16_ritems = nullptr;
  int32_t* m16_rcount = nullptr;
  double* m16_tpart = nullptr;
  // symmetric multi-RHS (8-vector chunks): B' items over the U box panels, T1 / Y1
  bool m_sym_ok = false;
  AItem* m_b1items = nullptr;
  int64_t m_n_b1items = 0;
  RItem* m_b1ritems = nullptr;
  int32_t* m_b1rcount = nullptr;
  double *m_b1tpart = nullptr, *m_t1 = nullptr, *m_y1 = nullptr;
  double* d_ynear = nullptr;              // [3n] near-field P2P slots (p2p_sym_kernel)
  // stored near field for 16-vector chunks (Alg. 1 l.5: the dense self / edge-sharer blocks
  // of every served leaf, column-major mp x ncolp per leaf at nf_off[leaf - leaf_begin])
  int nf_state = 0;                       // 0 not built, 1 built, -1 skipped (memory)
  bool nf_enabled = true;                 // set_diag "multi_stored_near"
  double* d_snf = nullptr;
  int64_t* d_snf_off = nullptr;
  int64_t nf_values = 0;
  double* d_yfar = nullptr;               // [served] low-rank part (stage B output)
  cudaStream_t hi_stream = nullptr;       // stages A, B (high priority)
  cudaStream_t aux_stream = nullptr;      // P2P (low priority), concurrent with A and B
  cudaStream_t copy_stream = nullptr;     // host <-> device copies of host-pointer calls
  cudaEvent_t ev_copy0 = nullptr, ev_copy1 = nullptr;
  // stream-ordered host-buffer matvecs (hodlr2d_matvec_async): H2D and D2H on their own
  // streams (the two copy engines), double-buffered device x / y so call k + 1's H2D and
  // call k - 1's D2H run under call k's kernels
  cudaStream_t as_h2d = nullptr, as_d2h = nullptr;
  double* as_x[2] = {nullptr, nullptr};
  double* as_y[2] = {nullptr, nullptr};
  cudaEvent_t as_xin[2] = {nullptr, nullptr}, as_xfree[2] = {nullptr, nullptr};
  cudaEvent_t as_ydone[2] = {nullptr, nullptr}, as_yfree[2] = {nullptr, nullptr};
  int64_t as_calls = 0;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_far = nullptr;
  // near-field placement on directed single-pass matvecs (apply.cu place_pick): beside stage A
  // (0, default) or beside stage B (1); -1: chosen by timing matvec calls 1-2 (A) against 3-4 (B)
  int p2p_place = 0, place_calls = 0;
  cudaEvent_t place_ev[4][2] = {};
  // P2P classes (generic CTA leaves, warp leaves of 3 / 2 rows per lane) fork from aux_stream
  // onto their own low-priority streams so their under-filled grids overlap
  cudaStream_t p2p_side[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_p2p_fork = nullptr, ev_p2p_side[3] = {nullptr, nullptr, nullptr};
  // diagnostics switches of the matvec: read once from the environment at
  // build, changeable per handle with hodlr2d_set_diag (never per call from the environment)
  bool diag_p2p_serial = false, diag_p2p_onestream = false, diag_dual_norow = false;
  bool diag_copy_stream = true;
  bool multi_repl = true;       // multi-RHS on-the-fly log near field on the replicated table (set_diag "multi_log_table")
  bool list_repl = false;       // adaptive near field on the replicated log table (pick_list_table)
  int diag_p2p_list_ctas = 1;   // adaptive near field beside the streams: CTAs per SM (H2D_P2P_LIST_CTAS)
  // near-field kernel id (kp.id, or kLogSafe when a near pair has a subnormal r^2)
  int p2p_kid = 0;
  // pinned host staging of pageable caller buffers (0: inputs, 1: outputs)
  void* pin[2] = {nullptr, nullptr};
  size_t pin_bytes[2] = {0, 0};
  // matvec work buffers
  double* d_xtree = nullptr;              // [n]
  double* d_ybuf = nullptr;               // [n] staging for host y
  double* d_xbuf = nullptr;               // [n] staging for host x
  // stats
  double tree_seconds = 0, aca_seconds = 0, pack_seconds = 0, build_seconds = 0;
  int64_t truncated = 0;
  // timing
  int timing = 0;
  std::vector<cudaEvent_t> ev_pool;
  int64_t ev_used = 0;
  int64_t ev_base = 0;
  int64_t timed_count = 0;
  double stage_ms[H2D_NUM_STAGES] = {};
  // allocations
  std::vector<void*> allocs;
  size_t device_bytes = 0;

  int64_t box_begin(int l, int64_t b) const {
    return leaf_start[(size_t)(b << (2 * (kappa - l)))];
  }
  int64_t box_end(int l, int64_t b) const {
    return leaf_start[(size_t)((b + 1) << (2 * (kappa - l)))];
  }
  bool row_box_active(int l, int64_t b) const {
    return box_begin(l, b) < row_end && box_end(l, b) > row_begin;
  }
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    H2D_CUDA(cudaMalloc(&p, count * sizeof(T)));
    allocs.push_back(p);
    device_bytes += count * sizeof(T);
    return static_cast<T*>(p);
  }
  void release(void* p);
  ~Handle();
};

// ------------------------------------------------------------------ host drivers
void build_tree(Handle& h, const double* d_points);              // tree.cu (G1-G4)
void build_lists(Handle& h);                                      // tree.cu (G5)
void build_adaptive(Handle& h);                                   // tree.cu (R24 leaves)
void build_adaptive_near(Handle& h);                              // tree.cu (R24 near field)
void run_aca(Handle& h);                                          // aca.cu (G6) + pack (G7)
// Pack the given per-block factor sources of one level into panels (apply.cu).
void pack_level(Handle& h, Level& L, const std::vector<const double*>& srcU,
                const std::vector<const double*>& srcV);
void finalize_schedule(Handle& h);                                // apply.cu
// Copy block e of level l out of the panels to host arrays (U m x r, V n x r, col-major).
void unpack_block(Handle& h, int l, int64_t e, int* m, int* n, int* r, double* U, double* V);
// gather: H2D_ORDER_LOCAL with a communicator — x_tree holds only the served rows when the
// call starts; the local stage-A items run before the all-gather completes (comm.cu)
void matvec_tree(Handle& h, const double* d_xtree, double* d_y, int order_out,
                 int64_t y_row0, bool gather = false);            // apply.cu (S7-S9)
// comm.cu (S11 behind the ABI)
void comm_init(Handle& h);
void comm_destroy(Handle& h);
void comm_unique_id(unsigned char* id);
int comm_kind(const Handle& h);   // 0 none, 1 NCCL, 2 host callback
void comm_gather_start(Handle& h, const double* d_xl, double* d_xtree);
void comm_gather_exchange(Handle& h);
cudaEvent_t comm_gather_finish(Handle& h, double* d_xtree, cudaStream_t st);
void permute_in(Handle& h, const double* d_x, double* d_xtree);   // apply.cu (S10)
// per-matvec CUDA events (timing mode): 0 start, 1 after input permute/unpad (caller
// stream); 2 after stage A, 3 after stage B (high-priority stream); 4 after joining the
// P2P, 5 end = after the combine epilogue (caller stream); 6/7 P2P (aux stream)
constexpr int kEventsPerMatvec = 8;
void begin_matvec_timing(Handle& h);
void mark_after_input(Handle& h);
void unpad_gathered(Handle& h, const double* d_xg, double* d_xtree);  // apply.cu (S11 epilogue)
void matvec_multi(Handle& h, const double* d_X, double* d_Y, int nrhs, int order);  // multi.cu
void gmres_solve(Handle& h, const double* d_b, double* d_x, double tol, int restart, int max_iter,
                 int* iters, double* relres);                             // gmres.cu

}  // namespace h2d
