// S11 behind the C ABI: the one x all-gather of the multi-GPU matvec (the
// paper's parallel HODLR2D distributes the matvec over processes with OpenMPI, §6, its
// static schedule and load model Eq. eq:par P:1256-1266).
//
// Rank g serves TREE rows [row_begin, row_end) (Morton ranges, capi.cu set_partition).  A
// matvec in H2D_ORDER_LOCAL takes only that slice of x; the library
//   1. places it in its own slot of a padded [world x gather_stride] buffer and in x_tree,
//   2. all-gathers the slots (ncclAllGather on the handle's communicator, in place, on a
//      high-priority comm stream — or, for hosts without NCCL between the ranks (tests of
//      several ranks on one GPU), through a caller-supplied host all-gather callback),
//   3. runs the stage-A items whose column box lies in the local range while the gather is
//      in flight, then unpads the other ranks' slots and runs the rest of S7-S9.
// NCCL is resolved at run time (dlopen of libnccl.so.2: the copy PyTorch already loaded, else
// the system one), so the library has no link-time NCCL dependency and loads without it.
#include <dlfcn.h>
#include <nccl.h>   // types and enums only; every function goes through the dlsym table

#include <cstring>

#include "h2d_internal.cuh"

namespace h2d {

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*MemFree)(void*) = nullptr;
  ncclResult_t (*CommRegister)(const ncclComm_t, void*, size_t, void**) = nullptr;
  ncclResult_t (*CommDeregister)(const ncclComm_t, void*) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi load_nccl() {
  NcclApi a;
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) {
    const char* e = dlerror();
    a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
    return a;
  }
  auto sym = [&](const char* name) { return dlsym(lib, name); };
  a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
  a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
  a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
  a.AllGather = (decltype(a.AllGather))sym("ncclAllGather");
  a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
  a.MemAlloc = (decltype(a.MemAlloc))sym("ncclMemAlloc");          // optional (NCCL >= 2.19)
  a.MemFree = (decltype(a.MemFree))sym("ncclMemFree");
  a.CommRegister = (decltype(a.CommRegister))sym("ncclCommRegister");
  a.CommDeregister = (decltype(a.CommDeregister))sym("ncclCommDeregister");
  a.CommGetAsyncError = (decltype(a.CommGetAsyncError))sym("ncclCommGetAsyncError");
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.GetErrorString;
  if (!a.ok) a.why = "libnccl.so.2 lacks ncclGetUniqueId / ncclCommInitRank / ncclAllGather";
  return a;
}

NcclApi& nccl() {
  static NcclApi api = load_nccl();
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error{H2D_ENCCL, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?")};
}

// x_tree[rows[r] + i] = xg[r * stride + i] for every rank r != skip (the local slot is
// already in place and may be read concurrently by the local stage-A items).
__global__ void unpad_remote_kernel(const double* __restrict__ xg, const int64_t* __restrict__ rows,
                                    int world, int skip, int64_t stride, int64_t n, double* __restrict__ xt) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    int r = 0;
    while (r + 1 < world && rows[r + 1] <= s) ++r;
    if (r != skip) xt[s] = xg[r * stride + (s - rows[r])];
  }
}

}  // namespace

struct Comm {
  int world = 1, rank = 0;
  ncclComm_t nc = nullptr;          // NCCL mode
  void* reg = nullptr;              // ncclCommRegister handle of gbuf
  bool gbuf_nccl = false;           // gbuf from ncclMemAlloc
  hodlr2d_allgather_fn fn = nullptr;  // host-staged mode
  void* ctx = nullptr;
  double* gbuf = nullptr;           // [world * stride] padded gather buffer (device)
  double* h_send = nullptr;         // [stride]          pinned (host-staged mode)
  double* h_recv = nullptr;         // [world * stride]  pinned (host-staged mode)
  cudaStream_t cs = nullptr;        // comm / copy stream (high priority)
  cudaEvent_t ev_in = nullptr, ev_gathered = nullptr, ev_xready = nullptr;
  ~Comm() {
    if (cs) cudaStreamSynchronize(cs);
    if (nc && reg && nccl().CommDeregister) nccl().CommDeregister(nc, reg);
    if (gbuf) {
      if (gbuf_nccl) nccl().MemFree(gbuf);
      else cudaFree(gbuf);
    }
    if (nc) nccl().CommDestroy(nc);
    if (h_send) cudaFreeHost(h_send);
    if (h_recv) cudaFreeHost(h_recv);
    for (cudaEvent_t e : {ev_in, ev_gathered, ev_xready})
      if (e) cudaEventDestroy(e);
    if (cs) cudaStreamDestroy(cs);
  }
};

int comm_kind(const Handle& h) { return !h.comm ? 0 : h.comm->nc ? 1 : 2; }

void comm_destroy(Handle& h) {
  delete h.comm;
  h.comm = nullptr;
}

void comm_unique_id(unsigned char* id) {
  if (!nccl().ok) throw Error{H2D_ENCCL, nccl().why};
  ncclUniqueId u;
  nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == H2D_COMM_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id, &u, sizeof(u));
}

// Called once at the end of the build when the options carry a communicator.
void comm_init(Handle& h) {
  const hodlr2d_options& o = h.opts;
  if (!o.nccl_id && !o.allgather) return;
  if (h.rank_rows.empty()) throw Error{H2D_EINVAL, "a communicator needs the world/rank partition (row_end <= 0)"};
  auto* c = new Comm();
  h.comm = c;
  c->world = o.world;
  c->rank = o.rank;
  int lo = 0, hi = 0;
  H2D_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  H2D_CUDA(cudaStreamCreateWithPriority(&c->cs, cudaStreamNonBlocking, hi));
  for (cudaEvent_t* e : {&c->ev_in, &c->ev_gathered, &c->ev_xready})
    H2D_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  const size_t bytes = (size_t)std::max<int64_t>(1, h.gather_stride) * (size_t)o.world * sizeof(double);
  if (o.nccl_id) {
    if (!nccl().ok) throw Error{H2D_ENCCL, nccl().why};
    ncclUniqueId u;
    std::memcpy(&u, o.nccl_id, sizeof(u));
    nccl_check(nccl().CommInitRank(&c->nc, o.world, u, o.rank), "ncclCommInitRank");
    // gather buffer from NCCL's allocator and registered with the communicator, so NCCL can
    // take its zero-copy / NVLS paths over NVSwitch; plain cudaMalloc if either is missing
    void* p = nullptr;
    if (nccl().MemAlloc && nccl().MemAlloc(&p, bytes) == ncclSuccess) {
      c->gbuf_nccl = true;
    } else {
      H2D_CUDA(cudaMalloc(&p, bytes));
    }
    c->gbuf = (double*)p;
    if (nccl().CommRegister && nccl().CommRegister(c->nc, p, bytes, &c->reg) != ncclSuccess) c->reg = nullptr;
  } else {
    c->fn = o.allgather;
    c->ctx = o.allgather_ctx;
    H2D_CUDA(cudaMalloc(&c->gbuf, bytes));
    H2D_CUDA(cudaMallocHost(&c->h_send, (size_t)std::max<int64_t>(1, h.gather_stride) * sizeof(double)));
    H2D_CUDA(cudaMallocHost(&c->h_recv, bytes));
  }
  H2D_CUDA(cudaMemset(c->gbuf, 0, bytes));
}

// Step 1-2 (before the local stage-A launch): the local slice d_xl (device, rows
// row_begin..row_end in TREE order) goes into x_tree and into its slot; NCCL mode enqueues
// the in-place all-gather on the comm stream, ordered after the caller's stream.
void comm_gather_start(Handle& h, const double* d_xl, double* d_xtree) {
  Comm* c = h.comm;
  // failure detection: an error NCCL raised asynchronously on this communicator (a peer
  // that died, a network fault) surfaces here as H2D_ENCCL instead of a hang in the gather
  if (c->nc && nccl().CommGetAsyncError) {
    ncclResult_t ae = ncclSuccess;
    nccl_check(nccl().CommGetAsyncError(c->nc, &ae), "ncclCommGetAsyncError");
    if (ae != ncclSuccess && ae != ncclInProgress) nccl_check(ae, "NCCL asynchronous error on the communicator");
  }
  const int64_t rows = h.row_end - h.row_begin;
  double* slot = c->gbuf + (int64_t)c->rank * h.gather_stride;
  if (rows > 0) {
    H2D_CUDA(cudaMemcpyAsync(d_xtree + h.row_begin, d_xl, rows * 8, cudaMemcpyDeviceToDevice, h.stream));
    H2D_CUDA(cudaMemcpyAsync(slot, d_xl, rows * 8, cudaMemcpyDeviceToDevice, h.stream));
  }
  H2D_CUDA(cudaEventRecord(c->ev_in, h.stream));
  H2D_CUDA(cudaStreamWaitEvent(c->cs, c->ev_in, 0));
  if (c->nc) {
    nccl_check(nccl().AllGather(slot, c->gbuf, (size_t)h.gather_stride, ncclFloat64, c->nc, c->cs), "ncclAllGather");
    H2D_CUDA(cudaEventRecord(c->ev_gathered, c->cs));
  } else if (rows > 0) {
    H2D_CUDA(cudaMemcpyAsync(c->h_send, d_xl, rows * 8, cudaMemcpyDeviceToHost, c->cs));
  }
}

// Step 2, host-staged mode (after the local launches, so they run during the exchange):
// wait for the local slice on the host, exchange through the callback, upload the slots.
void comm_gather_exchange(Handle& h) {
  Comm* c = h.comm;
  if (c->nc) return;
  H2D_CUDA(cudaStreamSynchronize(c->cs));
  const int64_t rows = h.row_end - h.row_begin;
  for (int64_t i = rows; i < h.gather_stride; ++i) c->h_send[i] = 0.0;   // padding
  const int rc = c->fn(c->h_send, c->h_recv, (size_t)h.gather_stride * sizeof(double), c->ctx);
  if (rc != 0) throw Error{H2D_ENCCL, "host all-gather callback failed (" + std::to_string(rc) + ")"};
  H2D_CUDA(cudaMemcpyAsync(c->gbuf, c->h_recv, (size_t)h.gather_stride * c->world * sizeof(double),
                           cudaMemcpyHostToDevice, c->cs));
  H2D_CUDA(cudaEventRecord(c->ev_gathered, c->cs));
}

// Step 3: stream st waits for the gathered slots and unpads the other ranks' rows into
// x_tree; returns the event recorded after the unpad (x_tree complete).
cudaEvent_t comm_gather_finish(Handle& h, double* d_xtree, cudaStream_t st) {
  Comm* c = h.comm;
  H2D_CUDA(cudaStreamWaitEvent(st, c->ev_gathered, 0));
  if (c->world > 1) {
    const int blocks = (int)std::min<int64_t>((h.n + 255) / 256, (int64_t)h.num_sms * 8);
    unpad_remote_kernel<<<blocks, 256, 0, st>>>(c->gbuf, h.d_rank_rows, c->world, c->rank, h.gather_stride, h.n,
                                                d_xtree);
    H2D_LAUNCH_CHECK();
  }
  H2D_CUDA(cudaEventRecord(c->ev_xready, st));
  return c->ev_xready;
}

}  // namespace h2d
