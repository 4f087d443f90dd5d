// C ABI of the B200 HODLR2D library (include/hodlr2d.h): handle lifecycle, build
// orchestration (Alg. 1), matvec entry points (Alg. 2), factor
// interchange file (R11), statistics and stage timing.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <fstream>
#include <new>
#include <thread>

#include "h2d_internal.cuh"

namespace h2d {

static thread_local std::string g_last_error;

void set_error(int code, const std::string& msg) {
  (void)code;
  g_last_error = msg;
}

void Handle::release(void* p) {
  if (!p) return;
  auto it = std::find(allocs.begin(), allocs.end(), p);
  if (it != allocs.end()) {
    allocs.erase(it);
    cudaFree(p);
  }
}

Handle::~Handle() {
  cudaStreamSynchronize(stream);
  comm_destroy(*this);
  for (void* p : pin)
    if (p) cudaFreeHost(p);
  for (void* p : allocs) cudaFree(p);
  for (auto e : ev_pool) cudaEventDestroy(e);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (ev_far) cudaEventDestroy(ev_far);
  if (aux_stream) cudaStreamDestroy(aux_stream);
  for (int k = 0; k < 3; ++k) {
    if (p2p_side[k]) cudaStreamDestroy(p2p_side[k]);
    if (ev_p2p_side[k]) cudaEventDestroy(ev_p2p_side[k]);
  }
  if (ev_p2p_fork) cudaEventDestroy(ev_p2p_fork);
  if (hi_stream) cudaStreamDestroy(hi_stream);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (ev_b1) cudaEventDestroy(ev_b1);
  for (auto& pe : place_ev)
    for (cudaEvent_t e : pe)
      if (e) cudaEventDestroy(e);
  if (ev_copy0) cudaEventDestroy(ev_copy0);
  if (ev_copy1) cudaEventDestroy(ev_copy1);
  if (as_h2d) cudaStreamSynchronize(as_h2d);
  if (as_d2h) cudaStreamSynchronize(as_d2h);
  if (as_h2d) cudaStreamDestroy(as_h2d);
  if (as_d2h) cudaStreamDestroy(as_d2h);
  for (int k = 0; k < 2; ++k) {
    for (cudaEvent_t e : {as_xin[k], as_xfree[k], as_ydone[k], as_yfree[k]})
      if (e) cudaEventDestroy(e);
  }
}

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Host <-> device copies of the host-pointer paths run on a dedicated non-blocking stream,
// event-ordered with the work stream: a single pinned H2D on the legacy default stream was
// measured at 12.8 GB/s vs 54 GB/s on a non-default stream (tools/copy_probe.py, 8 MB).
static void copy_stream_init(Handle& h) {
  if (h.copy_stream) return;
  H2D_CUDA(cudaStreamCreateWithFlags(&h.copy_stream, cudaStreamNonBlocking));
  H2D_CUDA(cudaEventCreateWithFlags(&h.ev_copy0, cudaEventDisableTiming));
  H2D_CUDA(cudaEventCreateWithFlags(&h.ev_copy1, cudaEventDisableTiming));
}

static bool is_pinned_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Host memcpy in up to 8 threads (pageable staging: one thread moves ~5-10 GB/s).
static void par_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t kMin = (size_t)1 << 20;
  const int nt = (int)std::min<size_t>(8, std::max<size_t>(1, bytes / kMin));
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (bytes / nt + 63) & ~(size_t)63;
  for (int t = 0; t < nt; ++t) {
    const size_t o = (size_t)t * per;
    if (o >= bytes) break;
    th.emplace_back([=] { std::memcpy((char*)dst + o, (const char*)src + o, std::min(per, bytes - o)); });
  }
  for (auto& t : th) t.join();
}

// Library-owned pinned staging buffer of at least `bytes` (pageable caller buffers): the
// previous copy through it has completed when this returns.
static void* pinned_stage(Handle& h, int which, size_t bytes) {
  if (h.copy_stream) H2D_CUDA(cudaStreamSynchronize(h.copy_stream));
  H2D_CUDA(cudaStreamSynchronize(h.stream));
  if (h.pin_bytes[which] < bytes) {
    if (h.pin[which]) cudaFreeHost(h.pin[which]);
    h.pin[which] = nullptr;
    H2D_CUDA(cudaMallocHost(&h.pin[which], bytes));
    h.pin_bytes[which] = bytes;
  }
  return h.pin[which];
}

// dst (device) <- src (host), ordered after the work already queued on the work stream and
// before everything queued on it afterwards.  Pageable src is staged through the handle's
// pinned buffer (SURVEY §8(b) ownership: the library stages host pointers).
static void h2d_ordered(Handle& h, void* dst, const void* src, size_t bytes) {
  if (bytes && !is_pinned_host(src)) {
    void* st = pinned_stage(h, 0, bytes);
    par_memcpy(st, src, bytes);
    src = st;
  }
  if (!h.diag_copy_stream) {   // H2D_COPY_STREAM=0: copies on the work stream (diagnostics)
    H2D_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h.stream));
    return;
  }
  copy_stream_init(h);
  H2D_CUDA(cudaEventRecord(h.ev_copy0, h.stream));
  H2D_CUDA(cudaStreamWaitEvent(h.copy_stream, h.ev_copy0, 0));
  H2D_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h.copy_stream));
  H2D_CUDA(cudaEventRecord(h.ev_copy1, h.copy_stream));
  H2D_CUDA(cudaStreamWaitEvent(h.stream, h.ev_copy1, 0));
}

// dst (host) <- src (device) after the work queued on the work stream; returns when done.
// Pageable dst: through the handle's pinned buffer, then a host copy.
static void d2h_ordered_sync(Handle& h, void* dst, const void* src, size_t bytes) {
  if (bytes && !is_pinned_host(dst)) {
    void* st = pinned_stage(h, 1, bytes);
    d2h_ordered_sync(h, st, src, bytes);
    par_memcpy(dst, st, bytes);
    return;
  }
  if (!h.diag_copy_stream) {
    H2D_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h.stream));
    H2D_CUDA(cudaStreamSynchronize(h.stream));
    return;
  }
  copy_stream_init(h);
  H2D_CUDA(cudaEventRecord(h.ev_copy0, h.stream));
  H2D_CUDA(cudaStreamWaitEvent(h.copy_stream, h.ev_copy0, 0));
  H2D_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h.copy_stream));
  H2D_CUDA(cudaStreamSynchronize(h.copy_stream));
}

static int depth_rule(int64_t n, int leaf_size) {  // R1
  int k = 0;
  while ((double)leaf_size * std::ldexp(1.0, 2 * k) < (double)n) ++k;
  return k;
}

// Release factor panels and the matvec schedule (before re-packing).
static void clear_factors(Handle& h) {
  for (int l = 1; l <= h.kappa; ++l) {
    Level& L = h.levels[(size_t)l];
    h.release(L.U); L.U = nullptr;
    h.release(L.V); L.V = nullptr;
    h.release(L.d_ucolbase); L.d_ucolbase = nullptr;
    h.release(L.d_uoff); L.d_uoff = nullptr;
    h.release(L.Ub); L.Ub = nullptr;
  }
  for (void* q : {(void*)h.d_t1, (void*)h.d_udst, (void*)h.d_b1items, (void*)h.d_b1ritems, (void*)h.d_b1rcount,
                  (void*)h.d_b1tpart})
    h.release(q);
  h.d_t1 = h.d_b1tpart = nullptr;
  h.d_udst = h.d_b1rcount = nullptr;
  h.d_b1items = nullptr;
  h.d_b1ritems = nullptr;
  h.n_b1items = 0;
  h.n_b1big = 0;
  for (void* q : {(void*)h.m_aitems, (void*)h.m_ritems, (void*)h.m_rcount, (void*)h.m_tpart, (void*)h.m_xm,
                  (void*)h.m_iperm, (void*)h.m_t, (void*)h.m_yfar, (void*)h.m_ynear})
    h.release(q);
  h.m_aitems = nullptr; h.m_ritems = nullptr; h.m_rcount = nullptr; h.m_tpart = nullptr;
  h.m_xm = h.m_t = h.m_yfar = h.m_ynear = nullptr;
  h.m_iperm = nullptr;
  h.m_n_aitems = 0;
  for (void* q : {(void*)h.m_b1items, (void*)h.m_b1ritems, (void*)h.m_b1rcount, (void*)h.m_b1tpart, (void*)h.m_t1,
                  (void*)h.m_y1, (void*)h.m16_aitems, (void*)h.m16_ritems, (void*)h.m16_rcount, (void*)h.m16_tpart})
    h.release(q);
  h.m16_aitems = nullptr; h.m16_ritems = nullptr; h.m16_rcount = nullptr; h.m16_tpart = nullptr;
  h.m16_n_aitems = 0;
  h.m_b1items = nullptr; h.m_b1ritems = nullptr; h.m_b1rcount = nullptr;
  h.m_b1tpart = h.m_t1 = h.m_y1 = nullptr;
  h.m_n_b1items = 0;
  h.m_sym_ok = false;
  h.multi_ready = false;
  h.release(h.d_bitems); h.d_bitems = nullptr;
  h.release(h.d_blev); h.d_blev = nullptr;
  h.n_bitems = 0;
  h.release(h.d_aitems); h.d_aitems = nullptr;
  h.release(h.d_ritems); h.d_ritems = nullptr;
  h.release(h.d_rcount); h.d_rcount = nullptr;
  h.release(h.d_t); h.d_t = nullptr;
  h.release(h.d_vdst); h.d_vdst = nullptr;
  h.release(h.d_tpart); h.d_tpart = nullptr;
  h.n_aitems = h.n_ritems = 0;
  h.n_abig = h.n_bbig = 0;
}

// |I_X| of box (cx, cy) at level l: children of the parent and its edge sharers (inside the
// domain) that are not edge or vertex neighbours of X (Eq. eq:ilist closed form, R5).
static int ilist_count(int l, int cx, int cy) {
  const int px = cx >> 1, py = cy >> 1, pside = 1 << (l - 1);
  const int dxs[5] = {0, -1, 1, 0, 0}, dys[5] = {0, 0, 0, -1, 1};
  int cnt = 0;
  for (int k = 0; k < 5; ++k) {
    const int qx = px + dxs[k], qy = py + dys[k];
    if (qx < 0 || qy < 0 || qx >= pside || qy >= pside) continue;
    for (int c = 0; c < 4; ++c)
      if (std::abs(2 * qx + (c & 1) - cx) + std::abs(2 * qy + (c >> 1) - cy) >= 2) ++cnt;
  }
  return cnt;
}

static uint32_t compact_host(uint32_t v) {
  v &= 0x55555555u;
  v = (v | (v >> 1)) & 0x33333333u;
  v = (v | (v >> 2)) & 0x0F0F0F0Fu;
  v = (v | (v >> 4)) & 0x00FF00FFu;
  v = (v | (v >> 8)) & 0x0000FFFFu;
  return v;
}

// Contiguous Morton ranges of leaves cut at the quantiles of a per-leaf load (SURVEY §8(e),
// in the spirit of Eq. eq:par): w(L) = |L| (1 + sum_l |I_{X_l}|) over L's
// ancestors X_l — the rows of L times the blocks each of them meets, a geometric proxy of
// the factor bytes (ranks are unknown before ACA).  Boxes near the domain boundary have
// fewer partners, so equal point shares left the centre-facing ranks ~12 % heavier (C5).
// The cut before rank r is the first leaf whose load prefix reaches r / world of the total.
// Cut position of rank boundary r on the prefix sums pre[] of the per-leaf loads, snapped to
// a coarse box boundary when that costs little balance: a cut inside a level-l box makes
// both neighbouring ranks stream the whole V panels of that box's partners (stage A needs
// V^T x over every row of the column box), which is ~8 % of a rank's bytes for a level-2
// box at C5 (measured: the ranks cutting level-2 boxes read 50.5 vs 46.8 GB).  Tolerance:
// 3 % of a share at level 1, 4 % at level 2, 4x less per finer level.
static int64_t snapped_cut(const std::vector<double>& pre, int kappa, int world, int r) {
  const int64_t nleaf = (int64_t)pre.size() - 1;
  if (r <= 0) return 0;
  if (r >= world) return nleaf;
  const double share = pre[(size_t)nleaf] / world, target = share * r;
  const int64_t c = (int64_t)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
  for (int l = 1; l <= std::min(kappa, 5); ++l) {
    const int64_t B = (int64_t)1 << (2 * (kappa - l));
    const double tol = (l == 1 ? 0.03 : 0.04 / (double)((int64_t)1 << (2 * (l - 2)))) * share;
    const int64_t lo = c / B * B, hi = std::min(nleaf, lo + B);
    const int64_t sn = std::fabs(pre[(size_t)lo] - target) <= std::fabs(pre[(size_t)hi] - target) ? lo : hi;
    if (std::fabs(pre[(size_t)sn] - target) <= tol) return sn;
  }
  return std::min(c, nleaf);
}

static void partition_leaves(const int32_t* ls, int kappa, int world, int rank, int64_t* lb,
                             int64_t* le, const double* weights = nullptr) {
  const int64_t nleaf = (int64_t)1 << (2 * kappa);
  std::vector<double> pre((size_t)nleaf + 1, 0.0);
  if (weights) {   // measured loads (hodlr2d_leaf_costs summed over ranks)
    for (int64_t L = 0; L < nleaf; ++L) pre[(size_t)L + 1] = pre[(size_t)L] + std::max(0.0, weights[L]);
  } else {
    std::vector<std::vector<uint8_t>> cnt((size_t)kappa + 1);
    for (int l = 1; l <= kappa; ++l) {
      const int64_t nbox = (int64_t)1 << (2 * l);
      cnt[(size_t)l].resize((size_t)nbox);
      for (int64_t b = 0; b < nbox; ++b)
        cnt[(size_t)l][(size_t)b] =
            (uint8_t)ilist_count(l, (int)compact_host((uint32_t)b), (int)compact_host((uint32_t)b >> 1));
    }
    for (int64_t L = 0; L < nleaf; ++L) {
      int s = 1;
      for (int l = 1; l <= kappa; ++l) s += cnt[(size_t)l][(size_t)(L >> (2 * (kappa - l)))];
      pre[(size_t)L + 1] = pre[(size_t)L] + (double)(ls[L + 1] - ls[L]) * s;
    }
  }
  *lb = snapped_cut(pre, kappa, world, rank);
  *le = snapped_cut(pre, kappa, world, rank + 1);
}

static void set_partition(Handle& h) {
  const int64_t nleaf = (int64_t)1 << (2 * h.kappa);
  if (h.opts.row_end > 0) {
    // snap an explicit row range to leaf boundaries
    auto snap = [&](int64_t r) {
      return (int64_t)(std::lower_bound(h.leaf_start.begin(), h.leaf_start.end(), (int32_t)r) -
                       h.leaf_start.begin());
    };
    h.leaf_begin = std::min<int64_t>(snap(std::max<int64_t>(0, h.opts.row_begin)), nleaf);
    h.leaf_end = std::min<int64_t>(snap(std::min<int64_t>(h.n, h.opts.row_end)), nleaf);
    if (h.opts.row_end >= h.n) h.leaf_end = nleaf;
  } else {
    partition_leaves(h.leaf_start.data(), h.kappa, h.opts.world, h.opts.rank, &h.leaf_begin,
                     &h.leaf_end, h.opts.leaf_weights);
    // every rank's rows: layout of the padded all-gather (H2D_ORDER_GATHERED)
    h.rank_rows.assign((size_t)h.opts.world + 1, 0);
    for (int r = 0; r < h.opts.world; ++r) {
      int64_t lb = 0, le = 0;
      partition_leaves(h.leaf_start.data(), h.kappa, h.opts.world, r, &lb, &le, h.opts.leaf_weights);
      h.rank_rows[(size_t)r] = h.leaf_start[(size_t)lb];
      h.rank_rows[(size_t)r + 1] = h.leaf_start[(size_t)le];
      h.gather_stride = std::max<int64_t>(h.gather_stride, h.leaf_start[(size_t)le] - h.leaf_start[(size_t)lb]);
    }
    h.d_rank_rows = h.alloc<int64_t>(h.rank_rows.size());
    H2D_CUDA(cudaMemcpy(h.d_rank_rows, h.rank_rows.data(), h.rank_rows.size() * 8, cudaMemcpyHostToDevice));
  }
  h.row_begin = h.leaf_start[(size_t)h.leaf_begin];
  h.row_end = h.leaf_start[(size_t)h.leaf_end];
}

static void skip_factors(Handle& h) {
  for (int l = 1; l <= h.kappa; ++l) {
    Level& L = h.levels[(size_t)l];
    L.rank.assign((size_t)L.nblocks, -1);
    L.truncated.assign((size_t)L.nblocks, 0);
    std::vector<const double*> su((size_t)L.nblocks, nullptr), sv((size_t)L.nblocks, nullptr);
    pack_level(h, L, su, sv);
  }
}

static void do_matvec(Handle& h, const double* x, double* y, int order) {
  if (order != H2D_ORDER_ORIGINAL && order != H2D_ORDER_TREE && order != H2D_ORDER_GATHERED &&
      order != H2D_ORDER_LOCAL)
    throw Error{H2D_EINVAL, "bad order"};
  if (order == H2D_ORDER_LOCAL && !h.comm)
    throw Error{H2D_EINVAL, "LOCAL order needs a communicator (options.nccl_id or options.allgather)"};
  if (!x || !y) throw Error{H2D_EINVAL, "null x or y"};
  const bool part = h.row_begin != 0 || h.row_end != h.n;
  if (order == H2D_ORDER_ORIGINAL && part)
    throw Error{H2D_EINVAL, "ORIGINAL order needs a single-rank (full-range) handle"};
  if (order == H2D_ORDER_GATHERED && h.rank_rows.empty())
    throw Error{H2D_EINVAL, "GATHERED order needs a world/rank partition"};
  const int64_t xlen = order == H2D_ORDER_GATHERED ? h.gather_stride * h.opts.world
                     : order == H2D_ORDER_LOCAL  ? h.row_end - h.row_begin
                                                 : h.n;
  cudaStream_t s = h.stream;
  const bool xdev = is_device_ptr(x), ydev = is_device_ptr(y);
  const int64_t ylen = order == H2D_ORDER_ORIGINAL ? h.n : (h.row_end - h.row_begin);
  begin_matvec_timing(h);
  const double* xin = x;
  if (!xdev) {
    if (!h.d_xbuf) h.d_xbuf = h.alloc<double>(std::max<int64_t>(h.n, h.gather_stride * h.opts.world));
    h2d_ordered(h, h.d_xbuf, x, xlen * sizeof(double));
    xin = h.d_xbuf;
  }
  double* yout = y;
  if (!ydev) {
    if (!h.d_ybuf) h.d_ybuf = h.alloc<double>(h.n);
    yout = h.d_ybuf;
  }
  const double* xt = xin;
  if (order == H2D_ORDER_ORIGINAL) {
    permute_in(h, xin, h.d_xtree);
    xt = h.d_xtree;
  } else if (order == H2D_ORDER_GATHERED) {
    unpad_gathered(h, xin, h.d_xtree);
    xt = h.d_xtree;
  } else if (order == H2D_ORDER_LOCAL) {   // S11: the library gathers x itself (comm.cu)
    comm_gather_start(h, xin, h.d_xtree);
    xt = h.d_xtree;
  }
  mark_after_input(h);
  matvec_tree(h, xt, yout, order == H2D_ORDER_ORIGINAL ? H2D_ORDER_ORIGINAL : H2D_ORDER_TREE,
              h.row_begin, order == H2D_ORDER_LOCAL);
  if (h.timing) h.timed_count++;
  if (!ydev) {
    d2h_ordered_sync(h, y, yout, ylen * sizeof(double));
  } else if (!xdev) {
    H2D_CUDA(cudaStreamSynchronize(h.copy_stream ? h.copy_stream : s));  // x reusable on return
  }
  (void)s;
}

// Stream-ordered matvec on pinned host (or device) buffers: H2D of x on as_h2d, the matvec on
// the work stream, D2H of y on as_d2h, each ordered by events; returns once enqueued.  Device
// staging slot k & 1: call k's H2D waits until call k - 2's kernels no longer read its x
// slot, its kernels wait until call k - 2's D2H has drained its y slot.
static void matvec_async(Handle& h, const double* x, double* y, int order) {
  if (order != H2D_ORDER_ORIGINAL && order != H2D_ORDER_TREE && order != H2D_ORDER_GATHERED)
    throw Error{H2D_EINVAL, "async matvec: order must be ORIGINAL, TREE or GATHERED"};
  if (!x || !y) throw Error{H2D_EINVAL, "null x or y"};
  if (order == H2D_ORDER_ORIGINAL && (h.row_begin != 0 || h.row_end != h.n))
    throw Error{H2D_EINVAL, "ORIGINAL order needs a single-rank (full-range) handle"};
  if (order == H2D_ORDER_GATHERED && h.rank_rows.empty())
    throw Error{H2D_EINVAL, "GATHERED order needs a world/rank partition"};
  const bool xdev = is_device_ptr(x), ydev = is_device_ptr(y);
  if ((!xdev && !is_pinned_host(x)) || (!ydev && !is_pinned_host(y)))
    throw Error{H2D_EINVAL, "async matvec: x and y must be pinned host or device memory"};
  const int64_t xlen = order == H2D_ORDER_GATHERED ? h.gather_stride * h.opts.world : h.n;
  const int64_t ylen = order == H2D_ORDER_ORIGINAL ? h.n : (h.row_end - h.row_begin);
  if (!h.as_h2d) {
    H2D_CUDA(cudaStreamCreateWithFlags(&h.as_h2d, cudaStreamNonBlocking));
    H2D_CUDA(cudaStreamCreateWithFlags(&h.as_d2h, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k)
      for (cudaEvent_t* e : {&h.as_xin[k], &h.as_xfree[k], &h.as_ydone[k], &h.as_yfree[k]})
        H2D_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    // the first calls must not overtake work already queued on the caller's stream
    H2D_CUDA(cudaEventRecord(h.as_xfree[0], h.stream));
    H2D_CUDA(cudaEventRecord(h.as_xfree[1], h.stream));
  }
  const int sl = (int)(h.as_calls & 1);
  cudaStream_t s = h.stream;
  const double* xin = x;
  if (!xdev) {
    if (!h.as_x[sl]) h.as_x[sl] = h.alloc<double>(std::max<int64_t>(h.n, h.gather_stride * h.opts.world));
    H2D_CUDA(cudaStreamWaitEvent(h.as_h2d, h.as_xfree[sl], 0));
    H2D_CUDA(cudaMemcpyAsync(h.as_x[sl], x, xlen * sizeof(double), cudaMemcpyHostToDevice, h.as_h2d));
    H2D_CUDA(cudaEventRecord(h.as_xin[sl], h.as_h2d));
    H2D_CUDA(cudaStreamWaitEvent(s, h.as_xin[sl], 0));
    xin = h.as_x[sl];
  }
  double* yout = y;
  if (!ydev) {
    if (!h.as_y[sl]) h.as_y[sl] = h.alloc<double>(h.n);
    H2D_CUDA(cudaStreamWaitEvent(s, h.as_yfree[sl], 0));
    yout = h.as_y[sl];
  }
  begin_matvec_timing(h);
  const double* xt = xin;
  if (order == H2D_ORDER_ORIGINAL) {
    permute_in(h, xin, h.d_xtree);
    xt = h.d_xtree;
  } else if (order == H2D_ORDER_GATHERED) {
    unpad_gathered(h, xin, h.d_xtree);
    xt = h.d_xtree;
  }
  mark_after_input(h);
  matvec_tree(h, xt, yout, order == H2D_ORDER_ORIGINAL ? H2D_ORDER_ORIGINAL : H2D_ORDER_TREE, h.row_begin, false);
  if (h.timing) h.timed_count++;
  if (!xdev) H2D_CUDA(cudaEventRecord(h.as_xfree[sl], s));   // (TREE order reads x throughout)
  if (!ydev) {
    H2D_CUDA(cudaEventRecord(h.as_ydone[sl], s));
    H2D_CUDA(cudaStreamWaitEvent(h.as_d2h, h.as_ydone[sl], 0));
    H2D_CUDA(cudaMemcpyAsync(y, yout, ylen * sizeof(double), cudaMemcpyDeviceToHost, h.as_d2h));
    H2D_CUDA(cudaEventRecord(h.as_yfree[sl], h.as_d2h));
  }
  ++h.as_calls;
}

static void async_wait(Handle& h) {
  if (h.as_h2d) H2D_CUDA(cudaStreamSynchronize(h.as_h2d));
  H2D_CUDA(cudaStreamSynchronize(h.stream));
  if (h.as_d2h) H2D_CUDA(cudaStreamSynchronize(h.as_d2h));
}

// ---------------------------------------------------------------- factor interchange (R11)
struct FileHeader {
  int64_t N;
  int32_t kappa, kid;
  double tol, c, scale, shift, lo_x, lo_y, side;
  int32_t test_rank, reserved;
};

static void load_factors(Handle& h, const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Error{H2D_EFACTORS, std::string("cannot open ") + path};
  char magic[8];
  f.read(magic, 8);
  if (!f || std::memcmp(magic, "H2DFAC01", 8) != 0) throw Error{H2D_EFACTORS, "bad magic"};
  FileHeader hd{};
  f.read((char*)&hd.N, 8);
  f.read((char*)&hd.kappa, 4);
  f.read((char*)&hd.kid, 4);
  double d[7];
  f.read((char*)d, 56);
  f.read((char*)&hd.test_rank, 4);
  f.read((char*)&hd.reserved, 4);
  if (!f) throw Error{H2D_EFACTORS, "truncated header"};
  if (hd.N != h.n || hd.kappa != h.kappa)
    throw Error{H2D_EFACTORS, "file N/kappa do not match the handle"};
  if ((hd.reserved == 1) != h.adaptive)   // R11 / R24: the adaptive tree's block lists differ
    throw Error{H2D_EFACTORS, "file and handle disagree on the adaptive tree (depth = -3)"};
  std::vector<int32_t> fperm((size_t)hd.N), perm((size_t)h.n);
  f.read((char*)fperm.data(), hd.N * 4);
  H2D_CUDA(cudaMemcpy(perm.data(), h.d_perm, h.n * 4, cudaMemcpyDeviceToHost));
  if (fperm != perm) throw Error{H2D_EFACTORS, "file permutation does not match the handle's tree"};
  clear_factors(h);
  h.truncated = 0;
  h.pair_failed = false;
  for (auto& Lv : h.levels) { h.release(Lv.Pr); Lv.Pr = nullptr; Lv.pairs.clear(); }
  std::vector<char> discard((size_t)1 << 20);
  for (int l = 1; l <= h.kappa; ++l) {
    Level& L = h.levels[(size_t)l];
    int64_t nb = 0;
    f.read((char*)&nb, 8);
    if (!f || nb != L.nblocks) throw Error{H2D_EFACTORS, "block count mismatch at level " + std::to_string(l)};
    std::vector<double> host;
    std::vector<int64_t> uo((size_t)nb, -1), vo((size_t)nb, -1);
    L.rank.assign((size_t)nb, -1);
    L.truncated.assign((size_t)nb, 0);
    for (int64_t X = 0; X < L.nbox; ++X) {
      const int64_t m = h.box_end(l, X) - h.box_begin(l, X);
      const bool keep = h.row_box_active(l, X);
      for (int32_t e = L.off[(size_t)X]; e < L.off[(size_t)X + 1]; ++e) {
        const int64_t Y = L.col[(size_t)e];
        const int64_t n = h.box_end(l, Y) - h.box_begin(l, Y);
        int32_t r = 0;
        f.read((char*)&r, 4);
        // r = -1: block not stored by a row-restricted file (R11); fine unless served here
        if (!f || r < -1) throw Error{H2D_EFACTORS, "bad rank"};
        if (r == -1 && keep)
          throw Error{H2D_EFACTORS, "file lacks block " + std::to_string(e) + " of level " + std::to_string(l) +
                                        ", whose rows this handle serves"};
        const size_t cnt = r > 0 ? (size_t)r * (size_t)(m + n) : 0;
        if (keep) {
          L.rank[(size_t)e] = r;
          uo[(size_t)e] = (int64_t)host.size();
          vo[(size_t)e] = (int64_t)host.size() + (int64_t)r * m;
          size_t o = host.size();
          host.resize(o + cnt);
          f.read((char*)(host.data() + o), cnt * 8);
        } else {   // read and drop (no seek: the file may be a pipe from the producer)
          size_t left = cnt * 8;
          while (left > 0 && f) {
            const size_t k = std::min(left, discard.size());
            f.read(discard.data(), (std::streamsize)k);
            left -= k;
          }
        }
        if (!f) throw Error{H2D_EFACTORS, "truncated factors at level " + std::to_string(l)};
      }
    }
    double* d = nullptr;
    H2D_CUDA(cudaMalloc(&d, std::max<size_t>(1, host.size()) * 8));
    if (!host.empty()) H2D_CUDA(cudaMemcpy(d, host.data(), host.size() * 8, cudaMemcpyHostToDevice));
    std::vector<const double*> su((size_t)nb, nullptr), sv((size_t)nb, nullptr);
    for (int64_t e = 0; e < nb; ++e)
      if (uo[(size_t)e] >= 0) { su[(size_t)e] = d + uo[(size_t)e]; sv[(size_t)e] = d + vo[(size_t)e]; }
    pack_level(h, L, su, sv);
    H2D_CUDA(cudaFree(d));
  }
  finalize_schedule(h);
}

static void extract_block(Handle& h, int l, int64_t e, int* m, int* n, int* r, double* U, double* V) {
  unpack_block(h, l, e, m, n, r, U, V);
}

}  // namespace h2d

using namespace h2d;

struct hodlr2d_s {
  Handle h;
};

#define H2D_TRY try {
#define H2D_CATCH                                                   \
  }                                                                 \
  catch (const Error& err) {                                        \
    set_error(err.code, err.msg);                                   \
    return err.code;                                                \
  }                                                                 \
  catch (const std::bad_alloc&) {                                   \
    set_error(H2D_ENOMEM, "host allocation failed");               \
    return H2D_ENOMEM;                                              \
  }                                                                 \
  catch (const std::exception& ex) {                                \
    set_error(H2D_ECUDA, ex.what());                                \
    return H2D_ECUDA;                                               \
  }

extern "C" {

void hodlr2d_default_options(hodlr2d_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->c = 1.0;
  o->scale = 1.0;
  o->shift = 0.0;
  o->box_side = 0.0;
  o->depth = -1;
  o->max_rank = 128;
  o->aca_consecutive = 3;
  o->aca_trim = 3;
  o->test_rank = 1;
  o->stream = nullptr;
  o->world = 1;
  o->rank = 0;
  o->row_begin = 0;
  o->row_end = 0;
  o->aca_scratch_bytes = 0;
  o->timing = 0;
  o->skip_aca = 0;
}

int hodlr2d_build(const double* points, int64_t n, int kernel_id, int leaf_size, double aca_tol,
                  hodlr2d_t* out) {
  hodlr2d_options o;
  hodlr2d_default_options(&o);
  return hodlr2d_build_ex(points, n, kernel_id, leaf_size, aca_tol, &o, out);
}

int hodlr2d_build_ex(const double* points, int64_t n, int kernel_id, int leaf_size, double aca_tol,
                     const hodlr2d_options* opts, hodlr2d_t* out) {
  if (out) *out = nullptr;
  hodlr2d_s* H = nullptr;
  H2D_TRY
  if (!out || !points || !opts) throw Error{H2D_EINVAL, "null argument"};
  if (n < 1) throw Error{H2D_EINVAL, "n < 1"};
  if (n > INT32_MAX) throw Error{H2D_EINVAL, "n >= 2^31 not supported"};
  if (leaf_size < 1) throw Error{H2D_EINVAL, "leaf_size < 1"};
  if (!(aca_tol > 0.0 && aca_tol < 1.0)) throw Error{H2D_EINVAL, "aca_tol not in (0, 1)"};
  if (kernel_id != H2D_KERNEL_LOG && kernel_id != H2D_KERNEL_IMQ && kernel_id != H2D_KERNEL_ONE_OVER_R &&
      kernel_id != H2D_KERNEL_RBF_PHI1 && kernel_id != H2D_KERNEL_RBF_PHI2 &&
      kernel_id != H2D_KERNEL_TEST_LOWRANK)
    throw Error{H2D_EINVAL, "unknown kernel_id"};
  if (kernel_id == H2D_KERNEL_IMQ && !(opts->c > 0.0)) throw Error{H2D_EINVAL, "IMQ needs c > 0"};
  if ((kernel_id == H2D_KERNEL_RBF_PHI1 || kernel_id == H2D_KERNEL_RBF_PHI2) && !(opts->c > 0.0))
    throw Error{H2D_EINVAL, "RBF kernels need a = c > 0"};
  if (kernel_id == H2D_KERNEL_RBF_PHI1 && opts->c == 1.0)
    throw Error{H2D_EINVAL, "phi_1 needs a != 1 (log a = 0)"};
  if (opts->depth < -3) throw Error{H2D_EINVAL, "depth < -3"};
  if (opts->depth == -3 && (opts->world > 1 || opts->row_end > 0))
    throw Error{H2D_EINVAL, "the adaptive tree (depth = -3) supports single-rank handles only"};
  if (opts->max_rank < 1 || opts->aca_consecutive < 1 || opts->aca_trim < 0 ||
      opts->aca_trim > opts->aca_consecutive)
    throw Error{H2D_EINVAL, "bad ACA options"};
  if (opts->world < 1 || opts->rank < 0 || opts->rank >= opts->world)
    throw Error{H2D_EINVAL, "bad world/rank"};
  if (!std::isfinite(opts->scale) || !std::isfinite(opts->shift)) throw Error{H2D_EINVAL, "non-finite scale/shift"};
  double t0 = now_s();
  H = new hodlr2d_s();
  Handle& h = H->h;
  h.opts = *opts;
  h.stream = (cudaStream_t)opts->stream;
  H2D_CUDA(cudaGetDevice(&h.device));
  h.kernel_id = kernel_id;
  h.leaf_size = leaf_size;
  h.tol = aca_tol;
  h.n = n;
  h.kp.id = kernel_id;
  h.kp.inv_c2 = kernel_id == H2D_KERNEL_IMQ ? 1.0 / (opts->c * opts->c) : 0.0;
  h.kp.a = opts->c;
  h.kp.a2 = opts->c * opts->c;
  h.kp.inv_log_a = kernel_id == H2D_KERNEL_RBF_PHI1 ? 1.0 / std::log(opts->c) : 0.0;
  h.kp.inv_phi1_den = kernel_id == H2D_KERNEL_RBF_PHI1 ? 1.0 / (opts->c * std::log(opts->c) - 1.0) : 0.0;
  h.kp.scale = opts->scale;
  h.kp.shift = opts->shift;
  h.kp.test_rank = opts->test_rank;
  h.kappa = opts->depth >= 0 ? opts->depth : depth_rule(n, leaf_size);
  if (h.kappa > 15) throw Error{H2D_EINVAL, "depth > 15"};
  if (h.kappa > H2D_MAX_LEVELS) throw Error{H2D_EINVAL, "depth > H2D_MAX_LEVELS"};
  h.timing = opts->timing;
  {   // diagnostics switches, read once here
    auto env_is = [](const char* name, int v) { const char* e = getenv(name); return e && atoi(e) == v; };
    h.diag_p2p_serial = env_is("H2D_P2P_SERIAL", 1);
    if (getenv("H2D_P2P_PLACE")) h.p2p_place = std::max(-1, std::min(1, atoi(getenv("H2D_P2P_PLACE"))));
    h.diag_p2p_onestream = env_is("H2D_P2P_ONESTREAM", 1);
    h.diag_dual_norow = getenv("H2D_DUAL_NOROW") != nullptr;
    h.diag_copy_stream = !env_is("H2D_COPY_STREAM", 0);
    if (const char* e = getenv("H2D_P2P_LIST_CTAS")) h.diag_p2p_list_ctas = std::max(1, std::min(3, atoi(e)));
  }
  const double* d_pts = points;
  double* tmp = nullptr;
  if (!is_device_ptr(points)) {
    H2D_CUDA(cudaMallocAsync(&tmp, n * 2 * sizeof(double), h.stream));
    H2D_CUDA(cudaMemcpyAsync(tmp, points, n * 2 * sizeof(double), cudaMemcpyHostToDevice, h.stream));
    d_pts = tmp;
  }
  build_tree(h, d_pts);
  if (opts->depth == -2 || opts->depth == -3) {
    // the paper's rule (Alg. 1 l.3; R22): deepen until no leaf holds more than
    // N_max = leaf_size points (the R1 depth is a lower bound)
    for (;;) {
      int32_t mx = 0;
      for (size_t b = 0; b + 1 < h.leaf_start.size(); ++b) mx = std::max(mx, h.leaf_start[b + 1] - h.leaf_start[b]);
      if (mx <= leaf_size) break;
      // R24: the adaptive tree stops at level 11 (its per-level structures are indexed by
      // the 4^l Morton grid); boxes of level 11 holding more than N_max points stay leaves
      if (opts->depth == -3 && h.kappa >= 11) break;
      if (h.kappa >= 15) throw Error{H2D_EINVAL, "no depth <= 15 keeps every leaf <= N_max"};
      for (void* q : {(void*)h.d_perm, (void*)h.d_px, (void*)h.d_py, (void*)h.d_leaf_start}) h.release(q);
      ++h.kappa;
      build_tree(h, d_pts);
    }
  }
  if (tmp) H2D_CUDA(cudaFreeAsync(tmp, h.stream));
  if (opts->depth == -3) {   // adaptive quadtree (R24) below R22's deepest level
    h.adaptive = true;
    build_adaptive(h);
  }
  build_lists(h);
  set_partition(h);
  if (h.adaptive) {   // single rank: every adaptive leaf is served
    h.leaf_begin = 0;
    h.leaf_end = (int64_t)h.lf_code.size();
    build_adaptive_near(h);
  }
  h.opts.leaf_weights = nullptr;   // caller-owned, read only by the partition above
  comm_init(h);                    // S11 communicator (collective over the world's ranks)
  h.opts.nccl_id = nullptr;        // caller-owned, read only by comm_init
  // symmetric apply (R23): symmetric build on a single-rank handle (the multi-rank row
  // partitions keep the directed panels; stage B' needs every row of a row box)
  // pair-local symmetric apply (pairs.cuh): symmetric builds on single-rank handles, with
  // H2D_PAIRAPPLY=1 (measured slower than the three-pass apply on C3 so far)
  {
    const char* e = getenv("H2D_PAIRAPPLY");
    const bool want = e ? atoi(e) != 0 : false;
    h.pair_wanted = want && opts->symmetric && h.row_begin == 0 && h.row_end == h.n && h.kappa >= 1;
  }
  // (multi-rank handles too: A' / B' run over the whole boxes of every pair that touches the
  // served rows, C' over the served leaves, the combine keeps the served rows)
  h.symapply = opts->symmetric && h.kappa >= 1 &&
               !(getenv("H2D_SYMAPPLY") && atoi(getenv("H2D_SYMAPPLY")) == 0);
  h.tree_seconds = now_s() - t0;
  if (opts->skip_aca) skip_factors(h); else run_aca(h);
  finalize_schedule(h);
  h.d_xtree = h.alloc<double>(n);
  H2D_CUDA(cudaStreamSynchronize(h.stream));
  h.build_seconds = now_s() - t0;
  *out = H;
  return h.truncated > 0 ? H2D_WTRUNC : H2D_OK;
  }
  catch (const Error& err) {
    delete H;
    set_error(err.code, err.msg);
    return err.code;
  }
  catch (const std::bad_alloc&) {
    delete H;
    set_error(H2D_ENOMEM, "host allocation failed");
    return H2D_ENOMEM;
  }
}

int hodlr2d_matvec(hodlr2d_t H, const double* x, double* y) {
  H2D_TRY
  if (!H) throw Error{H2D_EINVAL, "null handle"};
  do_matvec(H->h, x, y, H2D_ORDER_ORIGINAL);
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_matvec_ex(hodlr2d_t H, const double* x, double* y, int order) {
  H2D_TRY
  if (!H) throw Error{H2D_EINVAL, "null handle"};
  do_matvec(H->h, x, y, order);
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_matvec_async(hodlr2d_t H, const double* x, double* y, int order) {
  H2D_TRY
  if (!H) throw Error{H2D_EINVAL, "null handle"};
  matvec_async(H->h, x, y, order);
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_wait(hodlr2d_t H) {
  H2D_TRY
  if (!H) throw Error{H2D_EINVAL, "null handle"};
  async_wait(H->h);
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_matvec_multi(hodlr2d_t H, const double* X, double* Y, int nrhs, int order) {
  H2D_TRY
  if (!H || !X || !Y) throw Error{H2D_EINVAL, "null argument"};
  if (nrhs < 1) throw Error{H2D_EINVAL, "nrhs < 1"};
  Handle& h = H->h;
  if (order != H2D_ORDER_ORIGINAL && order != H2D_ORDER_TREE && order != H2D_ORDER_GATHERED &&
      order != H2D_ORDER_LOCAL)
    throw Error{H2D_EINVAL, "bad order"};
  if (order == H2D_ORDER_LOCAL && !h.comm)
    throw Error{H2D_EINVAL, "LOCAL order needs a communicator (options.nccl_id or options.allgather)"};
  if (order == H2D_ORDER_GATHERED && h.rank_rows.empty())
    throw Error{H2D_EINVAL, "GATHERED order needs a world/rank partition"};
  if (order == H2D_ORDER_LOCAL || h.adaptive) {
    // one vector at a time: the in-library gather (S11) and the adaptive tree (R24) run
    // through the single-vector matvec
    const int64_t rows = h.row_end - h.row_begin;
    const int64_t lx = order == H2D_ORDER_LOCAL ? rows : order == H2D_ORDER_GATHERED ? h.gather_stride * h.opts.world : h.n;
    const int64_t ly = order == H2D_ORDER_ORIGINAL ? h.n : rows;
    for (int k = 0; k < nrhs; ++k) do_matvec(h, X + (int64_t)k * lx, Y + (int64_t)k * ly, order);
    return H2D_OK;
  }
  cudaStream_t s = h.stream;
  const bool gathered = order == H2D_ORDER_GATHERED;
  const int64_t xlen = gathered ? h.gather_stride * h.opts.world : h.n;
  const int64_t ylen = order == H2D_ORDER_ORIGINAL ? h.n : h.row_end - h.row_begin;
  const bool xdev = is_device_ptr(X), ydev = is_device_ptr(Y);
  const double* dX = X;
  double* dY = Y;
  double *tx = nullptr, *ty = nullptr;
  if (!xdev) {
    H2D_CUDA(cudaMallocAsync(&tx, (size_t)nrhs * xlen * sizeof(double), s));
    h2d_ordered(h, tx, X, (size_t)nrhs * xlen * sizeof(double));
    dX = tx;
  }
  if (!ydev) {
    H2D_CUDA(cudaMallocAsync(&ty, (size_t)nrhs * ylen * sizeof(double), s));
    dY = ty;
  }
  double* tg = nullptr;   // GATHERED: the vectors unpadded into TREE order
  try {
    if (gathered) {
      H2D_CUDA(cudaMallocAsync(&tg, (size_t)nrhs * h.n * sizeof(double), s));
      for (int k = 0; k < nrhs; ++k) unpad_gathered(h, dX + (int64_t)k * xlen, tg + (int64_t)k * h.n);
      matvec_multi(h, tg, dY, nrhs, H2D_ORDER_TREE);
    } else {
      matvec_multi(h, dX, dY, nrhs, order);
    }
  } catch (...) {
    if (tx) cudaFreeAsync(tx, s);
    if (ty) cudaFreeAsync(ty, s);
    if (tg) cudaFreeAsync(tg, s);
    throw;
  }
  if (tg) H2D_CUDA(cudaFreeAsync(tg, s));
  if (!ydev) d2h_ordered_sync(h, Y, dY, (size_t)nrhs * ylen * sizeof(double));
  if (tx) H2D_CUDA(cudaFreeAsync(tx, s));
  if (ty) H2D_CUDA(cudaFreeAsync(ty, s));
  if (!ydev || !xdev) H2D_CUDA(cudaStreamSynchronize(s));
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_gmres(hodlr2d_t H, const double* b, double* x, double tol, int restart, int max_iter,
                  int* iters, double* rel_residual) {
  H2D_TRY
  if (!H || !b || !x) throw Error{H2D_EINVAL, "null argument"};
  Handle& h = H->h;
  // argument checks before any staging allocation (nothing to release on these errors)
  if (h.row_begin != 0 || h.row_end != h.n) throw Error{H2D_EINVAL, "GMRES needs a single-rank handle"};
  if (!(tol > 0.0) || restart < 1 || max_iter < 1) throw Error{H2D_EINVAL, "bad GMRES parameters"};
  if (restart > 65535) throw Error{H2D_EINVAL, "restart > 65535 (grid limit of the dot-product launch)"};
  cudaStream_t s = h.stream;
  const bool bdev = is_device_ptr(b), xdev = is_device_ptr(x);
  const double* db = b;
  double* dx = x;
  double *tb = nullptr, *tx = nullptr;
  if (!bdev) {
    H2D_CUDA(cudaMallocAsync(&tb, h.n * sizeof(double), s));
    h2d_ordered(h, tb, b, h.n * sizeof(double));
    db = tb;
  }
  if (!xdev) {
    H2D_CUDA(cudaMallocAsync(&tx, h.n * sizeof(double), s));
    dx = tx;
  }
  int its = 0;
  double rr = 0.0;
  try {
    gmres_solve(h, db, dx, tol, restart, max_iter, &its, &rr);
  } catch (...) {
    if (tb) cudaFreeAsync(tb, s);
    if (tx) cudaFreeAsync(tx, s);
    throw;
  }
  if (!xdev) d2h_ordered_sync(h, x, dx, h.n * sizeof(double));
  if (tb) H2D_CUDA(cudaFreeAsync(tb, s));
  if (tx) H2D_CUDA(cudaFreeAsync(tx, s));
  H2D_CUDA(cudaStreamSynchronize(s));
  if (iters) *iters = its;
  if (rel_residual) *rel_residual = rr;
  return rr < tol ? H2D_OK : H2D_WNOCONV;
  H2D_CATCH
}

int hodlr2d_get_info(hodlr2d_t H, hodlr2d_info* info) {
  H2D_TRY
  if (!H || !info) throw Error{H2D_EINVAL, "null argument"};
  Handle& h = H->h;
  std::memset(info, 0, sizeof(*info));
  info->n = h.n;
  info->kappa = h.kappa;
  info->world = h.opts.world;
  info->rank = h.opts.rank;
  info->row_begin = h.row_begin;
  info->row_end = h.row_end;
  info->leaf_begin = h.leaf_begin;
  info->leaf_end = h.leaf_end;
  info->box_lo[0] = h.lo[0];
  info->box_lo[1] = h.lo[1];
  info->box_side = h.side;
  int64_t uv = 0, vv = 0, built = 0, rsum = 0;
  int rmax = 0;
  for (int l = 1; l <= h.kappa; ++l) {
    const Level& L = h.levels[(size_t)l];
    info->blocks_per_level[l] = L.nblocks;
    for (int32_t r : L.rank) {
      if (r < 0) continue;
      ++built;
      rsum += r;
      rmax = std::max(rmax, r);
      info->rank_hist[std::min(r, 128)]++;
    }
    uv += L.u_values;
    vv += L.v_values;
  }
  info->blocks_built = built;
  info->rank_max = rmax;
  info->u_values = uv;
  info->v_values = vv;
  int64_t near = 0;
  if (h.adaptive) {   // R24: every served leaf's rows times its dense column ranges
    for (int64_t lf = h.leaf_begin; lf < h.leaf_end; ++lf)
      for (int64_t e = h.ad_nf_off[(size_t)lf]; e < h.ad_nf_off[(size_t)lf + 1]; ++e)
        near += (h.leaf_e(lf) - h.leaf_s(lf)) * h.ad_nf_rng[(size_t)(2 * e + 1)];
  }
  for (int64_t X = h.leaf_begin; X < h.leaf_end && !h.adaptive; ++X) {
    const int64_t m = h.leaf_start[(size_t)X + 1] - h.leaf_start[(size_t)X];
    for (int32_t e = h.nf_off[(size_t)X]; e < h.nf_off[(size_t)X + 1]; ++e) {
      const int32_t Y = h.nf_col[(size_t)e];
      near += m * (h.leaf_start[(size_t)Y + 1] - h.leaf_start[(size_t)Y]);
    }
  }
  info->near_pairs = near;
  info->p2p_pairs = (double)near;
  info->compression_ratio = ((double)(uv + vv) + (double)near) / ((double)h.n * (double)h.n);
  info->truncated = h.truncated;
  info->tree_seconds = h.tree_seconds;
  info->aca_seconds = h.aca_seconds;
  info->pack_seconds = h.pack_seconds;
  info->build_seconds = h.build_seconds;
  // algorithmic bytes: stage A reads V + x per chunk and writes t;
  // stage B reads U + t (+ tidx) + near-field points/x and writes y.
  const int64_t served = h.row_end - h.row_begin;
  // stage A: V panels once, x once, t (+ its destination index) written once.  stage B:
  // U panels once, t read once, ynear read once, y written once.  P2P: points + x + ynear.
  info->stageA_bytes = 8 * vv + 8 * (int64_t)h.n + 12 * h.t_len;
  info->stageB_bytes = 8 * uv + 8 * h.t_len + 16 * served;
  if (h.symapply) {
    // symmetric apply (R23): "stage A" = A' (first-side V box panels, x, t1 + its
    // destination index written) + B' (first-side U box panels, x, t1 read, t2 + udst, the
    // kappa y1 rows written); "stage B" = C' (second-side U leaf panels, t2) + the combine's
    // y1 / ynear / y traffic
    int64_t ub = 0;
    for (int l = 1; l <= h.kappa; ++l) ub += h.levels[(size_t)l].ub_values;
    info->stageA_bytes = 8 * vv + 8 * ub + 16 * (int64_t)h.n + 20 * h.t1_len + 12 * h.t_len +
                         8 * (int64_t)h.kappa * h.n;
    info->stageB_bytes = 8 * uv + 8 * h.t_len + 16 * served + 8 * (int64_t)h.kappa * served;
  }
  if (h.pairapply) {
    // pair apply: every pair's V and U once from HBM (the phase-3 V re-read is an L2 hit),
    // x read once, the y accumulator zeroed and reduced into (L2); "stage B" is empty
    info->stageA_bytes = 8 * h.pair_values + 8 * (int64_t)h.n + 8 * (int64_t)h.n;
    info->stageB_bytes = 16 * served;   // the combine's yacc read and y write
  }
  info->p2p_bytes = 24 * served + 8 * served;
  info->matvec_bytes = info->stageA_bytes + info->stageB_bytes + info->p2p_bytes;
  info->device_bytes = (int64_t)h.device_bytes;
  info->gather_stride = h.gather_stride;
  info->symmetric_apply = h.symapply ? 1 : 0;
  info->p2p_leaves[0] = h.n_p2p_warp;
  info->p2p_leaves[1] = h.n_p2p_fast;
  info->p2p_leaves[2] = h.n_p2p_gen;
  info->p2p_launches = (h.n_p2p_warp_rpl[0] > 0) + (h.n_p2p_warp_rpl[1] > 0) + (h.n_p2p_warp_rpl[2] > 0) +
                       (h.n_p2p_fast > 0) + (h.n_p2p_gen > 0) + (h.n_p2p_list > 0);
  info->adaptive = h.adaptive ? 1 : 0;
  info->n_leaves = h.adaptive ? (int64_t)h.lf_code.size() : ((int64_t)1 << (2 * h.kappa));
  info->small_items[0] = h.n_aitems - h.n_abig;
  info->small_items[1] = h.n_bitems - h.n_bbig;
  info->apply_launches = (h.n_abig > 0) + (h.n_aitems > h.n_abig) + (h.n_bbig > 0) + (h.n_bitems > h.n_bbig) +
                         (h.symapply && h.n_b1big > 0) + (h.symapply && h.n_b1items > h.n_b1big);
  if (h.pairapply) info->apply_launches = 1;
  info->pair_apply = h.pairapply ? 1 : 0;
  info->comm_kind = comm_kind(h);
  info->local_items[0] = h.n_abig_loc;
  info->local_items[1] = h.n_asmall_loc;
  info->stored_near_values = h.nf_state == 1 ? h.nf_values : 0;
  info->p2p_log_table = h.p2p_kid == kLogNoSelRepl ? 1 : h.p2p_kid == kLogNoSel ? 0 : -1;
  if (h.n_p2p_list > 0 && h.p2p_kid != kLogSafe && (h.kp.id == H2D_KERNEL_LOG || h.kp.id == H2D_KERNEL_RBF_PHI1))
    info->p2p_log_table = h.list_repl ? 1 : 0;
  (void)rsum;
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_copy_tree(hodlr2d_t H, int32_t* perm, int32_t* leaf_start) {
  H2D_TRY
  if (!H) throw Error{H2D_EINVAL, "null handle"};
  Handle& h = H->h;
  if (perm) H2D_CUDA(cudaMemcpy(perm, h.d_perm, h.n * 4, cudaMemcpyDeviceToHost));
  if (leaf_start) std::memcpy(leaf_start, h.leaf_start.data(), h.leaf_start.size() * 4);
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_copy_lists(hodlr2d_t H, int level, int32_t* off, int32_t* col) {
  H2D_TRY
  if (!H) throw Error{H2D_EINVAL, "null handle"};
  Handle& h = H->h;
  if (level < 0 || level > h.kappa) throw Error{H2D_EINVAL, "level out of range"};
  const int32_t* d_off = level == 0 ? h.d_nf_off : h.levels[(size_t)level].d_off;
  const int32_t* d_col = level == 0 ? h.d_nf_col : h.levels[(size_t)level].d_col;
  const int64_t nbox = (int64_t)1 << (2 * (level == 0 ? h.kappa : level));
  const int64_t tot = level == 0 ? h.nf_off[(size_t)nbox] : h.levels[(size_t)level].nblocks;
  // copy from the DEVICE arrays (what the kernels use)
  if (off) H2D_CUDA(cudaMemcpy(off, d_off, (nbox + 1) * 4, cudaMemcpyDeviceToHost));
  if (col && tot) H2D_CUDA(cudaMemcpy(col, d_col, tot * 4, cudaMemcpyDeviceToHost));
  return H2D_OK;
  H2D_CATCH
}

int64_t hodlr2d_num_blocks(hodlr2d_t H, int level) {
  if (!H || level < 0 || level > H->h.kappa) return -1;
  if (level == 0) return H->h.nf_off.empty() ? 0 : H->h.nf_off.back();
  return H->h.levels[(size_t)level].nblocks;
}

int hodlr2d_copy_ranks(hodlr2d_t H, int level, int32_t* ranks) {
  H2D_TRY
  if (!H || !ranks) throw Error{H2D_EINVAL, "null argument"};
  Handle& h = H->h;
  if (level < 1 || level > h.kappa) throw Error{H2D_EINVAL, "level out of range"};
  const Level& L = h.levels[(size_t)level];
  std::memcpy(ranks, L.rank.data(), L.rank.size() * 4);
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_copy_block(hodlr2d_t H, int level, int64_t e, int* m, int* n, int* r, double* U,
                       double* V) {
  H2D_TRY
  if (!H || !m || !n || !r) throw Error{H2D_EINVAL, "null argument"};
  Handle& h = H->h;
  if (level < 1 || level > h.kappa) throw Error{H2D_EINVAL, "level out of range"};
  if (e < 0 || e >= h.levels[(size_t)level].nblocks) throw Error{H2D_EINVAL, "block out of range"};
  extract_block(h, level, e, m, n, r, U, V);
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_load_factors(hodlr2d_t H, const char* path) {
  H2D_TRY
  if (!H || !path) throw Error{H2D_EINVAL, "null argument"};
  load_factors(H->h, path);
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_save_factors(hodlr2d_t H, const char* path) {
  H2D_TRY
  if (!H || !path) throw Error{H2D_EINVAL, "null argument"};
  Handle& h = H->h;
  if (h.row_begin != 0 || h.row_end != h.n) throw Error{H2D_EINVAL, "row-restricted handle"};
  std::ofstream f(path, std::ios::binary);
  if (!f) throw Error{H2D_EFACTORS, std::string("cannot open ") + path};
  f.write("H2DFAC01", 8);
  int64_t N = h.n;
  int32_t kap = h.kappa, kid = h.kernel_id, tr = h.opts.test_rank, res = h.adaptive ? 1 : 0;   // R11 / R24
  double c = h.kp.inv_c2 > 0 ? 1.0 / std::sqrt(h.kp.inv_c2) : h.opts.c;
  double d[7] = {h.tol, c, h.kp.scale, h.kp.shift, h.lo[0], h.lo[1], h.side};
  f.write((char*)&N, 8);
  f.write((char*)&kap, 4);
  f.write((char*)&kid, 4);
  f.write((char*)d, 56);
  f.write((char*)&tr, 4);
  f.write((char*)&res, 4);
  std::vector<int32_t> perm((size_t)h.n);
  H2D_CUDA(cudaMemcpy(perm.data(), h.d_perm, h.n * 4, cudaMemcpyDeviceToHost));
  f.write((char*)perm.data(), h.n * 4);
  for (int l = 1; l <= h.kappa; ++l) {
    const Level& L = h.levels[(size_t)l];
    int64_t nb = L.nblocks;
    f.write((char*)&nb, 8);
    std::vector<double> U, V;
    for (int64_t e = 0; e < nb; ++e) {
      int m, n, r;
      extract_block(h, l, e, &m, &n, &r, nullptr, nullptr);
      U.resize((size_t)m * r + 1);
      V.resize((size_t)n * r + 1);
      extract_block(h, l, e, &m, &n, &r, U.data(), V.data());
      int32_t rr = r;
      f.write((char*)&rr, 4);
      if (r) {
        f.write((char*)U.data(), (size_t)m * r * 8);
        f.write((char*)V.data(), (size_t)n * r * 8);
      }
    }
  }
  if (!f) throw Error{H2D_EFACTORS, "write failed"};
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_set_timing(hodlr2d_t H, int on) {
  if (!H) return H2D_EINVAL;
  H->h.timing = on ? 1 : 0;
  return H2D_OK;
}

int hodlr2d_stage_times(hodlr2d_t H, double* ms, int64_t* count, int reset) {
  H2D_TRY
  if (!H) throw Error{H2D_EINVAL, "null handle"};
  Handle& h = H->h;
  H2D_CUDA(cudaStreamSynchronize(h.stream));
  // kEventsPerMatvec events per matvec (see h2d_internal.cuh)
  static const int from[H2D_NUM_STAGES] = {0, 1, 2, 3, 4, 6};
  static const int to[H2D_NUM_STAGES] = {1, 2, 3, 4, 5, 7};
  double acc[H2D_NUM_STAGES] = {};
  const int64_t groups = h.ev_used / kEventsPerMatvec;
  for (int64_t g = 0; g < groups; ++g) {
    const size_t b = (size_t)(g * kEventsPerMatvec);
    for (int k = 0; k < H2D_NUM_STAGES; ++k) {
      float t = 0.f;
      H2D_CUDA(cudaEventElapsedTime(&t, h.ev_pool[b + from[k]], h.ev_pool[b + to[k]]));
      acc[k] += t;
    }
  }
  if (ms)
    for (int k = 0; k < H2D_NUM_STAGES; ++k) ms[k] = acc[k];
  if (count) *count = groups;
  if (reset) { h.ev_used = 0; h.timed_count = 0; }
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_destroy(hodlr2d_t H) {
  delete H;
  return H2D_OK;
}

const char* hodlr2d_last_error(void) { return g_last_error.c_str(); }

int64_t hodlr2d_copy_leaves(hodlr2d_t H, int32_t* level, int32_t* box) {
  if (!H) return -1;
  Handle& h = H->h;
  const int64_t n = h.adaptive ? (int64_t)h.lf_code.size() : ((int64_t)1 << (2 * h.kappa));
  for (int64_t lf = 0; lf < n; ++lf) {
    const int l = h.leaf_level(lf);
    if (level) level[lf] = l;
    if (box) box[lf] = (int32_t)(h.leaf_code(lf) >> (2 * (h.kappa - l)));
  }
  return n;
}

int hodlr2d_set_diag(hodlr2d_t H, const char* name, int value) {
  H2D_TRY
  if (!H || !name) throw Error{H2D_EINVAL, "null argument"};
  Handle& h = H->h;
  const std::string nm(name);
  if (nm == "p2p_serial") h.diag_p2p_serial = value != 0;
  else if (nm == "p2p_onestream") h.diag_p2p_onestream = value != 0;
  else if (nm == "p2p_place") {   // near field beside stage A (0) / stage B (1) / timed (-1)
    if (value < -1 || value > 1) throw Error{H2D_EINVAL, "p2p_place: -1, 0 or 1"};
    h.p2p_place = value;
    h.place_calls = 0;
  }
  else if (nm == "dual_norow") h.diag_dual_norow = value != 0;
  else if (nm == "copy_stream") h.diag_copy_stream = value != 0;
  else if (nm == "multi_stored_near") h.nf_enabled = value != 0;
  else if (nm == "multi_log_table") h.multi_repl = value != 0;   // 1: replicated 64-bin table
  else if (nm == "pair_apply") {   // symmetric handles: pair apply (1) or the three-pass apply (0)
    if (value && (!h.pair_wanted || h.pair_failed)) throw Error{H2D_EINVAL, "pair apply not built for this handle"};
    if (!value && !h.symapply && h.pairapply) throw Error{H2D_EINVAL, "no three-pass apply on this handle"};
    h.pairapply = value != 0;
  }
  else throw Error{H2D_EINVAL, "unknown diagnostics switch " + nm};
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_comm_unique_id(unsigned char* id) {
  H2D_TRY
  if (!id) throw Error{H2D_EINVAL, "null id"};
  comm_unique_id(id);
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_leaf_costs(hodlr2d_t H, double* costs) {
  H2D_TRY
  if (!H || !costs) throw Error{H2D_EINVAL, "null argument"};
  Handle& h = H->h;
  const int64_t nleaf = (int64_t)1 << (2 * h.kappa);
  for (int64_t L = 0; L < nleaf; ++L) costs[L] = 0.0;
  if (h.adaptive) throw Error{H2D_EINVAL, "leaf costs are defined for the balanced tree's partition"};
  for (int64_t L = h.leaf_begin; L < h.leaf_end; ++L) {
    const double rows = (double)(h.leaf_start[(size_t)L + 1] - h.leaf_start[(size_t)L]);
    double cols = 0.0;
    for (int l = 1; l <= h.kappa; ++l) {
      const Level& Lv = h.levels[(size_t)l];
      const int64_t X = L >> (2 * (h.kappa - l));
      if (!Lv.ucolbase.empty()) cols += Lv.ucolbase[(size_t)X + 1] - Lv.ucolbase[(size_t)X];
      if (!Lv.vR.empty()) cols += Lv.vR[(size_t)X];
    }
    costs[L] = 8.0 * rows * cols + 24.0 * rows;
  }
  return H2D_OK;
  H2D_CATCH
}

int hodlr2d_partition(const int32_t* leaf_start, int kappa, int world, int rank,
                      int64_t* leaf_begin, int64_t* leaf_end) {
  H2D_TRY
  // the same depth cap as the build (leaf_start must hold 4^kappa + 1 entries)
  if (!leaf_start || !leaf_begin || !leaf_end || kappa < 0 || kappa > 15 || world < 1 || rank < 0 ||
      rank >= world)
    throw Error{H2D_EINVAL, "bad partition arguments"};
  partition_leaves(leaf_start, kappa, world, rank, leaf_begin, leaf_end);
  return H2D_OK;
  H2D_CATCH
}

}  // extern "C"
