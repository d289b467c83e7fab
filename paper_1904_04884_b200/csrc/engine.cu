// Device-resident FISTA engine and the extern "C" boundary (include/holo_b200.h).
//
// The outer loop restates solver.py:254-379 (complex engine) on the host in
// C++; every O(volume) operation runs in the sm_100a kernels of kernels.cu.
// Per outer iteration the host reads back one small block of fp64 scalars.
//
// State layout in HBM (per rank, nzl local planes, P = ny*nx):
//   X[3]      nzl*P complex64  -- x_k, x_{k-1}, candidate (rotating slots)
//   S[3]      P complex64      -- sensor spectra A x of the three slots
//   scratch   nzl*P complex64  -- adjoint gradient / forward row-pass output
//   Spart     G*P complex64    -- per-group forward partial spectra
//   Bspec, R  P complex64      -- FFT(b) and the masked residual spectrum
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#ifdef HOLO_WITH_NCCL
#include <dlfcn.h>
#include <nccl.h>
#endif

#include "../../include/holo_b200.h"
#include "kernels.cuh"
#include <nvtx3/nvToolsExt.h>

namespace holo {

static thread_local std::string g_err;

struct Status {
  int code = HOLO_OK;
  static Status ok() { return Status(); }
};

#define HOLO_CUDA(expr)                                                                    \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      g_err = std::string(#expr) + ": " + cudaGetErrorString(_e);                          \
      return HOLO_ERR_CUDA;                                                                \
    }                                                                                      \
  } while (0)

#ifdef HOLO_WITH_NCCL
#define HOLO_NCCL(expr)                                                                    \
  do {                                                                                     \
    ncclResult_t _r = (expr);                                                              \
    if (_r != ncclSuccess) {                                                               \
      g_err = std::string(#expr) + ": " + ncclGetErrorString(_r);                          \
      return HOLO_ERR_NCCL;                                                                \
    }                                                                                      \
  } while (0)
#endif

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#ifdef HOLO_WITH_NCCL
// NCCL is resolved at run time (dlopen), not linked: in a process that already
// loaded PyTorch this binds to torch's bundled libnccl.so.2, and a process
// that never shards never loads NCCL at all.
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
      api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
      api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
      api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.getUniqueId && api.commInitRank && api.allReduce && api.commDestroy && api.getErrorString;
    }
  }
  return api;
}
#define ncclGetUniqueId(...) holo::nccl().getUniqueId(__VA_ARGS__)
#define ncclCommInitRank(...) holo::nccl().commInitRank(__VA_ARGS__)
#define ncclAllReduce(...) holo::nccl().allReduce(__VA_ARGS__)
#define ncclCommDestroy(...) holo::nccl().commDestroy(__VA_ARGS__)
#define ncclGetErrorString(...) holo::nccl().getErrorString(__VA_ARGS__)
#endif

template <class T>
static cudaError_t dalloc(T*& p, size_t count) {
  if (p) return cudaSuccess;
  cudaError_t e = cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1));
#ifdef HOLO_CHECKS
  // checked build: fresh buffers read as NaN / -1 until written
  if (!e) e = cudaMemset(p, 0xFF, sizeof(T) * std::max<size_t>(count, 1));
#endif
  return e;
}

// Per-kernel-class device timing with CUDA events on the launching stream
// (enabled by holo_profile_enable; harvested at each host sync point).
enum ProfKind { PK_ADJ_COLS = 0, PK_ADJ_ROWS, PK_PROX, PK_FWD_ROWS, PK_FWD_COLS, PK_SUM_GROUPS, PK_SENSOR, PK_REDUCE, PK_N };
static const char* kProfNames[PK_N] = {"adj_cols", "adj_rows", "prox", "fwd_rows",
                                       "fwd_cols", "sum_groups", "sensor", "reduce"};

struct Prof {
  bool on = false;
  unsigned mask = ~0u;  // classes that record (holo_profile_classes)
  bool cur = false;     // the open begin() recorded
  std::vector<cudaEvent_t> ev;
  std::vector<int> kind;
  int used = 0;
  double ms[PK_N] = {};
  long long cnt[PK_N] = {};
  void reset() {
    for (int i = 0; i < PK_N; ++i) { ms[i] = 0; cnt[i] = 0; }
  }
  cudaError_t begin(int k, cudaStream_t s) {
    // NVTX range per kernel class (header-only NVTX3: a no-op unless a tool
    // such as nsys / ncu --nvtx is attached)
    nvtxRangePushA(kProfNames[k]);
    cur = on && ((mask >> k) & 1u);
    if (!cur) return cudaSuccess;
    if ((int)kind.size() <= used) {
      cudaEvent_t a, b;
      cudaError_t e;
      if ((e = cudaEventCreate(&a))) return e;
      if ((e = cudaEventCreate(&b))) return e;
      ev.push_back(a);
      ev.push_back(b);
      kind.push_back(0);
    }
    kind[used] = k;
    return cudaEventRecord(ev[2 * used], s);
  }
  cudaError_t end(cudaStream_t s) {
    nvtxRangePop();
    if (!cur) return cudaSuccess;
    cur = false;
    cudaError_t e = cudaEventRecord(ev[2 * used + 1], s);
    ++used;
    return e;
  }
  // call after the stream has been synchronised
  cudaError_t harvest() {
    for (int i = 0; i < used; ++i) {
      float t = 0.f;
      cudaError_t e = cudaEventElapsedTime(&t, ev[2 * i], ev[2 * i + 1]);
      if (e) return e;
      ms[kind[i]] += t;
      cnt[kind[i]] += 1;
    }
    used = 0;
    return cudaSuccess;
  }
  ~Prof() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

#define PROF(kindv, s, call)                 \
  do {                                       \
    HOLO_CUDA(prof.begin((kindv), (s)));     \
    HOLO_CUDA(call);                         \
    HOLO_CUDA(prof.end((s)));                \
  } while (0)

// In-process rank group (holo_create_local_group): N engines on one GPU, each
// driven by its own host thread and stream, whose two collectives (spectrum and
// scalar allreduce) are an event-ordered device sum instead of NCCL.  Every
// member records an event after producing its buffer and blocks on the host
// until all members have; the last one makes its stream wait for all events,
// sums the buffers in rank order into each member's buffer, and records `done`,
// which every member's stream then waits on.  No kernel waits on another
// kernel: only stream/event ordering, so the sharded code path (plane ranges,
// partial spectra, scalar reductions, shared control decisions, per-rank COO)
// runs on one GPU exactly as it does under NCCL.
constexpr int kMaxGroup = 8;
struct GroupPtrs {
  const void* src[kMaxGroup];
  void* dst[kMaxGroup];
};
template <class T>
__global__ void k_group_sum(const GroupPtrs gp, int n, long long count) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
    T acc = static_cast<const T*>(gp.src[0])[i];
    for (int r = 1; r < n; ++r) acc += static_cast<const T*>(gp.src[r])[i];
    for (int r = 0; r < n; ++r) static_cast<T*>(gp.dst[r])[i] = acc;
  }
}

struct LocalGroup {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  void* buf[kMaxGroup] = {};
  cudaEvent_t ev[kMaxGroup] = {};
  cudaEvent_t done = nullptr;
  int refs = 0;
  ~LocalGroup() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (done) cudaEventDestroy(done);
  }
  cudaError_t init(int nn) {
    n = nn;
    cudaError_t e;
    for (int r = 0; r < n; ++r)
      if ((e = cudaEventCreateWithFlags(&ev[r], cudaEventDisableTiming))) return e;
    return cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
  }
  // stream barrier across members: every member's stream waits for every
  // member's work enqueued before the call (events; no kernel waits)
  cudaError_t barrier(int r, cudaStream_t s) {
    std::unique_lock<std::mutex> lk(m);
    cudaError_t e = cudaEventRecord(ev[r], s);
    if (e) return e;
    const long long my_gen = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my_gen; });
    }
    for (int i = 0; i < n; ++i)
      if ((e = cudaStreamWaitEvent(s, ev[i], 0))) return e;
    return cudaSuccess;
  }
  // sum over members of buf (count elements of T), in place on every member
  template <class T>
  cudaError_t allreduce(int r, T* b, long long count, cudaStream_t s) {
    std::unique_lock<std::mutex> lk(m);
    buf[r] = b;
    cudaError_t e = cudaEventRecord(ev[r], s);
    if (e) return e;
    const long long my_gen = gen;
    if (++arrived == n) {
      for (int i = 0; i < n; ++i)
        if ((e = cudaStreamWaitEvent(s, ev[i], 0))) return e;
      GroupPtrs gp{};
      for (int i = 0; i < n; ++i) gp.src[i] = gp.dst[i] = buf[i];
      const int threads = 256;
      const int blocks = (int)std::min<long long>((count + threads - 1) / threads, 148LL * 8);
      k_group_sum<T><<<std::max(blocks, 1), threads, 0, s>>>(gp, n, count);
      if ((e = cudaGetLastError())) return e;
      if ((e = cudaEventRecord(done, s))) return e;
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my_gen; });
      if ((e = cudaStreamWaitEvent(s, done, 0))) return e;
    }
    return cudaSuccess;
  }
};

// host scalar block (pinned) layout
enum Slot { SC_IP = 0, SC_DX2, SC_L1, SC_TV, SC_FAIL, SC_DEAD, SC_FY, SC_FNEW, SC_F0, SC_AUX, SC_N };

struct Engine {
  holo_geometry geom{};
  int device = 0, rank = 0, nranks = 1, kb = 0, ke = 0, nzl = 0;
  // Volume stack of the current solve.  Complex engine: nzs = nzl planes.
  // Packed real engine (real_nonnegative): x is real, so stack plane k holds
  // local real planes 2k (Re) and 2k+1 (Im), nzs = ceil(nzl / 2); the
  // transfer weights become U_k = c_2k + i c_2k+1 (c = Re H, see k_adj_cols),
  // the prox thresholds each part, and every volume kernel does half the
  // work.  With odd nzl the last Im part is a dummy plane held at zero (its
  // gradient is zeroed, so v, w and x_new stay 0 there).
  int nzs = 0;
  bool packed = false;
  void set_stack(bool pk) {
    packed = pk;
    nzs = pk ? (nzl + 1) / 2 : nzl;
  }
  bool dummy_part() const { return packed && (nzl & 1); }
  long long P = 0;
  cudaStream_t stream = nullptr;
  Plan plan;
#ifdef HOLO_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
  std::shared_ptr<LocalGroup> lgroup;  // in-process rank group (tests), else NCCL
  // peer-memory reduction of the forward spectrum (peer.cu): the rank group
  // always, NCCL ranks after holo_peer_import
  bool peer_on = false;
  PeerSet pset;
  float2* pr_inbox = nullptr;
  float2* pr_result = nullptr;
  unsigned long long* pr_flags = nullptr;
  unsigned* pr_counter = nullptr;  // [2] threadfence-reduction counters
  int* pr_err = nullptr;
  unsigned long long pr_epoch = 0;
  // a peer timeout leaves the ranks' epochs out of step: the handle is then
  // unusable (every later call fails with this message) until recreated
  bool peer_broken = false;
  std::vector<void*> pr_mapped;  // IPC mappings of the other ranks' buffers
  int ensure_peer_buffers() {
    if (pr_inbox) return HOLO_OK;
    const long long L = peer_slice(P, nranks);
    HOLO_CUDA(cudaMalloc(&pr_inbox, sizeof(float2) * (size_t)nranks * L));
    HOLO_CUDA(cudaMalloc(&pr_result, sizeof(float2) * (size_t)nranks * L));
    HOLO_CUDA(cudaMalloc(&pr_flags, sizeof(unsigned long long) * 2 * kMaxPeers));
    HOLO_CUDA(cudaMalloc(&pr_counter, sizeof(unsigned) * 2));
    HOLO_CUDA(cudaMalloc(&pr_err, sizeof(int)));
    HOLO_CUDA(cudaMemset(pr_flags, 0, sizeof(unsigned long long) * 2 * kMaxPeers));
    HOLO_CUDA(cudaMemset(pr_counter, 0, sizeof(unsigned) * 2));
    HOLO_CUDA(cudaMemset(pr_err, 0, sizeof(int)));
    pset.nranks = nranks;
    pset.rank = rank;
    pset.L = L;
    pset.inbox[rank] = pr_inbox;
    pset.result[rank] = pr_result;
    pset.flags[rank] = pr_flags;
    return HOLO_OK;
  }
  // S_out = sum over ranks of sum over plane groups of Spart (replaces
  // sum_groups + the spectrum allreduce)
  int peer_reduce(float2* S_out, int ngroups, cudaStream_t s) {
    const unsigned long long e = ++pr_epoch;
    const long long max_polls = 1LL << 26;  // ~20 s: a dead peer fails instead of hanging
    HOLO_CUDA(peer_scatter(Spart, ngroups, P, pset, e, pr_counter, s));
    if (lgroup) HOLO_CUDA(lgroup->barrier(rank, s));  // one GPU: no kernel may wait on another rank's
    HOLO_CUDA(peer_wait(pset, 0, e, max_polls, pr_err, s));
    HOLO_CUDA(peer_gather(P, pset, e, pr_counter + 1, s));
    if (lgroup) HOLO_CUDA(lgroup->barrier(rank, s));
    HOLO_CUDA(peer_wait(pset, 1, e, max_polls, pr_err, s));
    HOLO_CUDA(cudaMemcpyAsync(S_out, pr_result, sizeof(float2) * (size_t)P, cudaMemcpyDeviceToDevice, s));
    return HOLO_OK;
  }
  // volume buffers
  float2* X[3] = {nullptr, nullptr, nullptr};
  float2* scratch = nullptr;
  float2* Spart = nullptr;
  int groups = 1;
  // plane-sized buffers
  float2* S[3] = {nullptr, nullptr, nullptr};
  float2* Bspec = nullptr;
  float2* R = nullptr;
  double* b64 = nullptr;
  // reductions
  double* sens_part = nullptr;
  int sens_nblk = 0;
  double* scal = nullptr;       // device scalars [SC_N]
  double* h_scal = nullptr;     // pinned mirror
  double* prox_part = nullptr;  // [nzl][tpp][kProxParts]
  size_t prox_part_cap = 0;
  double* plane_out = nullptr;  // [nzl][4]
  int* new_fail = nullptr;      // [nzl]
  uint8_t* force_acc = nullptr; // [nzl]
  float4* tv_wside = nullptr;    // prox tvfix side rows [nzl][tiles][2][32]
  float* tv_bpart = nullptr;     // prox tvfix partials [nzl][3][tiles]
  size_t tvfix_cap = 0;          // tiles the two hold
  // sparsity-aware forward (solver.py:115-119): live[k] = 0 marks a stack
  // plane of the newest prox output that is all zero, so the forward row and
  // column passes skip it (HOLO_NO_PLANE_SKIP=1 turns the skipping off)
  uint8_t* live = nullptr;      // [nzl]
  bool plane_skip = std::getenv("HOLO_NO_PLANE_SKIP") == nullptr;
  float* fgp_beta = nullptr;
  int fgp_cap = 0;
  int fgp_inner = -1;  // depth whose momentum schedule fgp_beta holds
  // multi-pass FGP state (large T): v, 2 halves of (p,q) and (rp,rq), per-tile TV(v)
  float2* mp_v = nullptr;
  float4* mp_s = nullptr;
  float4* mp_r = nullptr;
  float* mp_tvv = nullptr;
  long long mp_cap = 0, mp_tiles = 0;
  // coo
  int* coo_counts = nullptr;
  long long* coo_offsets = nullptr;
  std::vector<int> h_counts;
  std::vector<long long> h_offsets;
  // device staging for host exports (grow-only)
  int32_t* coo_rows = nullptr;
  int32_t* coo_cols = nullptr;
  double2* coo_vals = nullptr;
  long long coo_cap = 0;
  // pinned double buffer for device -> pageable-host exports (lazy)
  void* stage_host[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  double real_sigma2 = -1.0;  // cached ||A_real||^2
  // results of the last solve
  int ix = 0;  // slot holding the solution
  bool have_solution = false;
  std::vector<double> history;
  holo_report last{};
  Prof prof;

  ~Engine() { release(); }

  void release() {
    for (auto& p : X) cudaFree(p);
    for (auto& p : S) cudaFree(p);
    cudaFree(scratch); cudaFree(Spart); cudaFree(Bspec); cudaFree(R); cudaFree(b64);
    cudaFree(sens_part); cudaFree(scal); cudaFreeHost(h_scal); cudaFree(prox_part);
    cudaFree(plane_out); cudaFree(new_fail); cudaFree(force_acc); cudaFree(live); cudaFree(fgp_beta);
    cudaFree(tv_wside); cudaFree(tv_bpart);
    cudaFree(coo_counts); cudaFree(coo_offsets);
    cudaFree(coo_rows); cudaFree(coo_cols); cudaFree(coo_vals);
    for (int i = 0; i < 2; ++i) {
      if (stage_host[i]) cudaFreeHost(stage_host[i]);
      if (stage_ev[i]) cudaEventDestroy(stage_ev[i]);
      stage_host[i] = nullptr;
      stage_ev[i] = nullptr;
    }
    cudaFree(mp_v); cudaFree(mp_s); cudaFree(mp_r); cudaFree(mp_tvv);
    for (void* m : pr_mapped) cudaIpcCloseMemHandle(m);
    pr_mapped.clear();
    cudaFree(pr_inbox); cudaFree(pr_result); cudaFree(pr_flags); cudaFree(pr_counter); cudaFree(pr_err);
    plan_free(plan);
#ifdef HOLO_WITH_NCCL
    if (comm) ncclCommDestroy(comm);
    comm = nullptr;
#endif
    if (stream) cudaStreamDestroy(stream);
    stream = nullptr;
  }

  // caller-supplied stream, CUDA convention: NULL is the legacy default stream
  static cudaStream_t st(void* s) { return (cudaStream_t)s; }

  int init(const holo_geometry& g, int dev, int r, int n) {
    geom = g;
    device = dev;
    rank = r;
    nranks = n;
    if (g.nx < 1 || g.ny < 1 || g.nz < 1) return fail(HOLO_ERR_INVALID, "voxel counts must be >= 1");
    if (!(g.pitch > 0) || !(g.dz > 0) || !(g.wavelength > 0)) return fail(HOLO_ERR_INVALID, "pitch, dz and wavelength must be positive");
    if (g.z0 < 0) return fail(HOLO_ERR_INVALID, "z0 must be nonnegative");
    if (!plan_supported(g.nx, g.ny))
      return fail(HOLO_ERR_UNSUPPORTED, "plane shape " + std::to_string(g.ny) + "x" + std::to_string(g.nx) +
                                            " unsupported: plane sides must lie in [8, 4096]");
    if (n < 1 || r < 0 || r >= n) return fail(HOLO_ERR_INVALID, "bad rank/nranks");
    // every rank owns >= 1 plane: an empty shard would launch zero-sized grids
    if (n > g.nz) return fail(HOLO_ERR_INVALID, "more ranks (" + std::to_string(n) + ") than planes (" +
                                                     std::to_string(g.nz) + ")");
    kb = (int)((long long)g.nz * r / n);
    ke = (int)((long long)g.nz * (r + 1) / n);
    nzl = ke - kb;
    set_stack(false);
    P = (long long)g.nx * g.ny;
    HOLO_CUDA(cudaSetDevice(dev));
    HOLO_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    HOLO_CUDA(plan_build(plan, g.nx, g.ny, g.nz, g.pitch, g.dz, g.z0, g.wavelength, stream));
    HOLO_CUDA(cudaMalloc(&scal, sizeof(double) * SC_N));
    HOLO_CUDA(cudaMallocHost(&h_scal, sizeof(double) * SC_N));
    sens_nblk = sensor_blocks(plan);
    HOLO_CUDA(cudaMalloc(&sens_part, sizeof(double) * std::max(sens_nblk, 2048)));
    return HOLO_OK;
  }

  int ensure_planes() {
    for (auto& p : S) HOLO_CUDA(dalloc(p, P));
    HOLO_CUDA(dalloc(Bspec, P));
    HOLO_CUDA(dalloc(R, P));
    HOLO_CUDA(dalloc(b64, P));
    return HOLO_OK;
  }

  int ensure_scratch() {
    HOLO_CUDA(dalloc(scratch, (size_t)nzl * P));
    groups = fwd_groups(plan, std::max(nzl, 1));
    HOLO_CUDA(dalloc(Spart, (size_t)groups * P));
    return ensure_planes();
  }

  int ensure_volume() {
    for (auto& p : X) HOLO_CUDA(dalloc(p, (size_t)nzl * P));
    HOLO_CUDA(dalloc(plane_out, (size_t)std::max(nzl, 1) * 4));
    HOLO_CUDA(dalloc(new_fail, std::max(nzl, 1)));
    HOLO_CUDA(dalloc(force_acc, std::max(nzl, 1)));
    HOLO_CUDA(dalloc(live, std::max(nzl, 1)));
    return ensure_scratch();
  }

  int ensure_prox(ProxArgs& a, int nplanes, int ny, int nx, int inner, cudaStream_t s) {
    prox_setup(a, ny, nx, inner);
    a.nplanes = nplanes;
    if (!prox_supported(ny, nx, inner))
      return fail(HOLO_ERR_UNSUPPORTED, "tv_inner_iters=" + std::to_string(inner) + " too deep for the single-pass prox tile");
    const size_t need = (size_t)std::max(nplanes, 1) * a.tiles_per_plane * kProxParts * std::max(1, (a.part_warps + 1) / 2);
    if (need > prox_part_cap) {
      cudaFree(prox_part);
      prox_part = nullptr;
      HOLO_CUDA(cudaMalloc(&prox_part, sizeof(double) * need));
      prox_part_cap = need;
    }
    a.part = prox_part;
    if (a.tvfix) {  // boundary-row statistics (k_prox_tvfix): w side rows + per-tile partials
      const size_t tiles = (size_t)std::max(nplanes, 1) * a.tiles_per_plane;
      if (tiles > tvfix_cap) {
        cudaFree(tv_wside);
        cudaFree(tv_bpart);
        tv_wside = nullptr;
        tv_bpart = nullptr;
        HOLO_CUDA(dalloc(tv_wside, tiles * 64));
        HOLO_CUDA(dalloc(tv_bpart, tiles * 3));
        tvfix_cap = tiles;
      }
      a.wside = tv_wside;
      a.bpart = tv_bpart;
    }
    if (a.pass_len) {  // multi-pass FGP state
      const long long n = (long long)std::max(nplanes, 1) * ny * nx;
      const long long tiles = (long long)std::max(nplanes, 1) * a.tiles_per_plane;
      if (n > mp_cap) {
        cudaFree(mp_v); cudaFree(mp_s); cudaFree(mp_r);
        mp_v = nullptr; mp_s = nullptr; mp_r = nullptr;
        HOLO_CUDA(cudaMalloc(&mp_v, sizeof(float2) * n));
        HOLO_CUDA(cudaMalloc(&mp_s, sizeof(float4) * 2 * n));
        HOLO_CUDA(cudaMalloc(&mp_r, sizeof(float4) * 2 * n));
        mp_cap = n;
      }
      if (tiles > mp_tiles) {
        cudaFree(mp_tvv);
        mp_tvv = nullptr;
        HOLO_CUDA(cudaMalloc(&mp_tvv, sizeof(float) * 2 * tiles));
        mp_tiles = tiles;
      }
      a.vbuf = mp_v;
      a.sbuf = mp_s;
      a.rbuf = mp_r;
      a.sstride = n;
      a.tvv = mp_tvv;
    }
    if (inner > fgp_cap) {
      cudaFree(fgp_beta);
      fgp_beta = nullptr;
      HOLO_CUDA(cudaMalloc(&fgp_beta, sizeof(float) * inner));
      fgp_cap = inner;
      fgp_inner = -1;
    }
    // data-independent FGP momentum (prox.py:132-133)
    std::vector<float> bt(inner);
    double t = 1.0;
    for (int i = 0; i < inner; ++i) {
      const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
      bt[i] = (float)((t - 1.0) / tn);
      t = tn;
    }
    for (int i = 0; i < inner && i < 16; ++i) a.fgpb[i] = bt[i];
    if (inner != fgp_inner) {  // once per depth: no stream sync on every attempt
      HOLO_CUDA(cudaMemcpyAsync(fgp_beta, bt.data(), sizeof(float) * inner, cudaMemcpyHostToDevice, s));
      HOLO_CUDA(cudaStreamSynchronize(s));  // bt is a stack buffer
      fgp_inner = inner;
    }
    a.fgp_beta = fgp_beta;
    return HOLO_OK;
  }

  // ---- collectives (no-ops on one rank) ----
  int allreduce_spec(float2* spec, cudaStream_t s) {
    if (nranks == 1) return HOLO_OK;
    if (lgroup) {
      HOLO_CUDA(lgroup->allreduce<float>(rank, reinterpret_cast<float*>(spec), P * 2, s));
      return HOLO_OK;
    }
#ifdef HOLO_WITH_NCCL
    HOLO_NCCL(ncclAllReduce(spec, spec, (size_t)P * 2, ncclFloat, ncclSum, comm, s));
    return HOLO_OK;
#else
    return fail(HOLO_ERR_UNSUPPORTED, "built without NCCL");
#endif
  }
  int allreduce_scalars(double* d, int n, cudaStream_t s) {
    if (nranks == 1) return HOLO_OK;
    if (lgroup) {
      HOLO_CUDA(lgroup->allreduce<double>(rank, d, n, s));
      return HOLO_OK;
    }
#ifdef HOLO_WITH_NCCL
    HOLO_NCCL(ncclAllReduce(d, d, n, ncclDouble, ncclSum, comm, s));
    return HOLO_OK;
#else
    return fail(HOLO_ERR_UNSUPPORTED, "built without NCCL");
#endif
  }

  // S_out = A x (spectrum, band mask not applied; allreduced over ranks)
  // skip (optional): per-plane live flags of x from prox_reduce
  int forward_spectrum(const float2* x, float2* S_out, cudaStream_t s, const uint8_t* skip = nullptr) {
    const int g = std::min(groups, fwd_groups(plan, std::max(nzs, 1)));  // (Spart holds `groups` partials)
    PROF(PK_FWD_ROWS, s, fft_rows(plan, x, scratch, (long long)nzs * geom.ny, false, 1.0f, s, skip, geom.ny));
    PROF(PK_FWD_COLS, s, fwd_cols(plan, scratch, Spart, nzs, kb, g, s, packed, skip));
    if (peer_on && nranks > 1) {  // fused group sum + reduce-scatter + all-gather over peer memory
      HOLO_CUDA(prof.begin(PK_SUM_GROUPS, s));
      int rc = peer_reduce(S_out, g, s);
      HOLO_CUDA(prof.end(s));
      return rc;
    }
    PROF(PK_SUM_GROUPS, s, sum_groups(plan, Spart, g, S_out, s));
    return allreduce_spec(S_out, s);
  }

  // scratch = 2 A^H r with R the masked residual spectrum
  int adjoint_grad(const float2* Rm, float scale, cudaStream_t s) {
    PROF(PK_ADJ_COLS, s, adj_cols(plan, Rm, scratch, nzs, kb, s, packed));
    PROF(PK_ADJ_ROWS, s, fft_rows(plan, scratch, scratch, (long long)nzs * geom.ny, true, scale / (float)P, s));
    // the dummy Im part of the last stack plane gets no gradient (stays 0)
    if (dummy_part()) HOLO_CUDA(zero_imag(scratch + (size_t)(nzs - 1) * P, P, s));
    return HOLO_OK;
  }

  int load_b(const double* b_dev, cudaStream_t s) {
    int rc = ensure_volume();
    if (rc) return rc;
    int nblk = 0;
    HOLO_CUDA(load_hologram(b_dev, Bspec, P, sens_part, &nblk, s));
    HOLO_CUDA(final_sum(sens_part, nblk, 1.0, scal + SC_F0, s));
    // Bspec = fft2(b)
    HOLO_CUDA(fft_rows(plan, Bspec, Bspec, geom.ny, false, 1.0f, s));
    HOLO_CUDA(fft_cols(plan, Bspec, Bspec, 1, false, 1.0f, s));
    return HOLO_OK;
  }

  int read_scalars(cudaStream_t s) {
    HOLO_CUDA(cudaMemcpyAsync(h_scal, scal, sizeof(double) * SC_N, cudaMemcpyDeviceToHost, s));
    int perr = 0;
    if (peer_on) HOLO_CUDA(cudaMemcpyAsync(&perr, pr_err, sizeof(int), cudaMemcpyDeviceToHost, s));
    HOLO_CUDA(cudaStreamSynchronize(s));
    if (perr) {
      peer_broken = true;
      return fail(HOLO_ERR_NCCL, "peer spectrum reduction: a rank did not arrive (timeout)");
    }
    HOLO_CUDA(prof.harvest());
    return HOLO_OK;
  }

  struct Attempt {
    int slot;
    double f_new, f_y, step, pen, ip, dx2;
  };

  // prox + reductions for one attempt, writes candidate into X[c]
  int prox_step(ProxArgs& a, cudaStream_t s) {
    PROF(PK_PROX, s, prox(a, s));
    HOLO_CUDA(prof.begin(PK_REDUCE, s));
    // sum |x_new| == 0 proves an all-zero plane when no nonzero pixel can add
    // an underflowed 0: real mode sums x itself; the complex soft threshold's
    // |x| term is >= 2^-24 tau_l1 for every surviving pixel, normal for
    // tau_l1 >= 1e-15 (prox_strip.cu epilogue, k_prox hypot in fp64)
    const int skip_ok = a.real_mode || a.tau_l1 >= 1e-15f;
    HOLO_CUDA(prox_reduce(a, a.tau_tv, a.tau_tv > 0.f, force_acc, plane_out, new_fail, s, live, skip_ok));
    HOLO_CUDA(plane_total(plane_out, new_fail, nzs, scal, s, live));
    HOLO_CUDA(prof.end(s));
    return allreduce_scalars(scal, SC_DEAD + 1, s);
  }

  int real_opnorm_value(double& out, cudaStream_t s) {
    if (real_sigma2 < 0) {
      HOLO_CUDA(real_opnorm(plan, geom.nz, scal + SC_AUX, s));
      if (int rc = read_scalars(s)) return rc;
      real_sigma2 = h_scal[SC_AUX];
    }
    out = real_sigma2;
    return HOLO_OK;
  }

  // solver.py:225-247: power iteration of A^H A from v0 (unit norm)
  int power_iteration(const float2* v0, int iters, bool real, double& out, cudaStream_t s) {
    if (peer_broken) return fail(HOLO_ERR_NCCL, "an earlier peer spectrum reduction timed out: recreate the handle");
    int rc = ensure_volume();
    if (rc) return rc;
    set_stack(false);  // the reference's start vector, one complex plane per real plane
    const long long n = (long long)nzl * P;
    counted_slot = -1;
    have_solution = false;
    if (n) HOLO_CUDA(cudaMemcpyAsync(X[0], v0, sizeof(float2) * n, cudaMemcpyDeviceToDevice, s));
    float2* v = X[0];
    if (real) HOLO_CUDA(vol_rescale(v, n, nullptr, 1, s));
    const int nb = vol_norm2_blocks(std::max(n, 1LL));
    double* part = nullptr;
    HOLO_CUDA(cudaMallocAsync(&part, sizeof(double) * nb, s));
    struct FreeOnExit {  // every return path, early errors included
      double*& p;
      cudaStream_t st;
      ~FreeOnExit() { if (p) cudaFreeAsync(p, st); }
    } free_part{part, s};
    double nrm = 1.0;
    for (int it = 0; it < iters; ++it) {
      if ((rc = forward_spectrum(v, S[0], s))) return rc;  // v may be scratch: consumed in place
      // spectrum of the real sensor field h = A v: m (S(f) + conj S(-f)) / 2
      HOLO_CUDA(sensor(plan, S[0], nullptr, 1.f, 0.f, nullptr, R, sens_part, s));
      if ((rc = adjoint_grad(R, 1.0f, s))) return rc;  // scratch = A^H h
      if (real) HOLO_CUDA(vol_rescale(scratch, n, nullptr, 1, s));
      HOLO_CUDA(cudaMemsetAsync(scal, 0, sizeof(double), s));
      if (n) {
        HOLO_CUDA(vol_norm2(scratch, n, part, s));
        HOLO_CUDA(final_sum(part, nb, 1.0, scal, s));
      }
      if ((rc = allreduce_scalars(scal, 1, s))) return rc;
      if ((rc = read_scalars(s))) return rc;
      nrm = std::sqrt(h_scal[0]);
      HOLO_CUDA(vol_rescale(scratch, n, scal, real ? 1 : 0, s));
      v = scratch;
    }
    HOLO_CUDA(cudaStreamSynchronize(s));
    out = nrm;
    return HOLO_OK;
  }

  // solver.py:297-327 iterate_from(y, step) with y = (1+beta) x - beta xp
  int iterate_from(int sx, int sxp, double beta, double step, const holo_solver_config& cfg, Attempt& out,
                   cudaStream_t s) {
    int rc;
    const bool mom = beta != 0.0;
    // residual spectrum at y (linearity: S_y = (1+beta) S_x - beta S_xp)
    HOLO_CUDA(prof.begin(PK_SENSOR, s));
    HOLO_CUDA(sensor(plan, S[sx], mom ? S[sxp] : nullptr, (float)(1.0 + beta), (float)(-beta), Bspec, R, sens_part, s));
    HOLO_CUDA(final_sum(sens_part, sens_nblk, 1.0 / (double)P, scal + SC_FY, s));
    HOLO_CUDA(prof.end(s));
    int c = 0;
    while (c == sx || c == sxp) ++c;
    double sigma2 = (double)geom.nz;  // ||A||^2, closed form (see holo_operator_norm)
    if (cfg.real_nonnegative && (rc = real_opnorm_value(sigma2, s))) return rc;
    for (;;) {
      ProxArgs a;
      if ((rc = ensure_prox(a, nzs, geom.ny, geom.nx, cfg.tv_inner_iters, s))) return rc;
      // gradient 2 A^H r_y into scratch (the forward pass below reuses scratch,
      // so a backtracking retry recomputes it)
      if ((rc = adjoint_grad(R, 2.0f, s))) return rc;
      a.x = X[sx];
      a.xp = X[sxp];
      a.grad = scratch;
      a.xnew = X[c];
      a.beta = (float)beta;
      a.step = (float)step;
      a.tau_l1 = (float)(step * cfg.lambda_l1);
      a.tau_tv = (float)(step * cfg.lambda_tv);
      a.lr_tv = a.tau_tv > 0.f ? (float)(1.0 / (8.0 * (step * cfg.lambda_tv))) : 0.f;
      a.real_mode = cfg.real_nonnegative ? 1 : 0;
      // ip / dx2 feed only the sufficient-decrease test, which is analytic below 1/(2 sigma^2)
      a.ipdx = (cfg.step_policy == HOLO_POLICY_BACKTRACKING && 2.0 * sigma2 * step > 1.0 + 1e-14) ? 1 : 0;
      HOLO_CUDA(cudaMemsetAsync(force_acc, 0, std::max(nzs, 1), s));
      if ((rc = prox_step(a, s))) return rc;
      // forward of the candidate (the adjoint scratch is consumed, reuse it)
      // and its data term, queued behind the prox without a host round trip:
      // the guard flag is read back together with f_new
      auto forward_fnew = [&]() -> int {
        int r2 = forward_spectrum(X[c], S[c], s, plane_skip ? live : nullptr);
        if (r2) return r2;
        HOLO_CUDA(prof.begin(PK_SENSOR, s));
        HOLO_CUDA(sensor(plan, S[c], nullptr, 1.f, 0.f, Bspec, nullptr, sens_part, s));
        HOLO_CUDA(final_sum(sens_part, sens_nblk, 1.0 / (double)P, scal + SC_FNEW, s));
        HOLO_CUDA(prof.end(s));
        return read_scalars(s);
      };
      if ((rc = forward_fnew())) return rc;
      if (plane_skip) last.skipped_planes += (long long)(h_scal[SC_DEAD] + 0.5);
      if (h_scal[SC_FAIL] > 0.5) {
        // guard fix-up: planes whose TV output was worse than its input take the
        // identity for that part (prox.py:138-147); rare, so the speculative
        // forward above is simply redone
        // the speculative forward's row pass overwrote the gradient in
        // scratch: recompute it (R, the residual spectrum at y, is intact)
        if ((rc = adjoint_grad(R, 2.0f, s))) return rc;
        do {
          last.guard_fixups += 1;
          ProxArgs f = a;
          f.force = force_acc;
          if ((rc = prox_step(f, s))) return rc;
          if ((rc = read_scalars(s))) return rc;
        } while (h_scal[SC_FAIL] > 0.5);
        if ((rc = forward_fnew())) return rc;
      }
      last.attempts += 1;
      out.slot = c;
      out.f_new = h_scal[SC_FNEW];
      out.f_y = h_scal[SC_FY];
      out.step = step;
      out.ip = h_scal[SC_IP];
      out.dx2 = h_scal[SC_DX2];
      // complex: lam1 sum|x| + lamTV (TV re + TV im); real engine: lam1 sum x + lamTV TV(x)
      // (x >= 0 and Im = 0 there, so the same two sums; solver.py:146-151 / 212-216)
      out.pen = cfg.lambda_l1 * h_scal[SC_L1] + (cfg.lambda_tv > 0 ? cfg.lambda_tv * h_scal[SC_TV] : 0.0);
      if (cfg.step_policy != HOLO_POLICY_BACKTRACKING) return HOLO_OK;
      // Sufficient-decrease test of solver.py:324-326.  With ||A||^2 = nz the
      // exact slack f_new - bound = ||A d||^2 - ||d||^2/(2 step) is <= 0 for
      // every step <= 1/(2 nz), so the reference (fp64, 1e-12 relative slack)
      // accepts; evaluating it in fp32 would only add rounding noise.
      if (2.0 * sigma2 * step <= 1.0 + 1e-14) return HOLO_OK;
      const double bound = out.f_y + out.ip + out.dx2 / (2.0 * step);
      if (out.f_new <= bound + 1e-12 * std::max(1.0, std::fabs(bound)) || step < 1e-30) return HOLO_OK;
      step *= cfg.bt_shrink;
    }
  }

  int counted_slot = -1;  // slot whose chunk counts/offsets are current (host + device)
  long long counted_total = 0;

  // the solution as one complex64 plane per local real plane: slot `slot`, or
  // for the packed real engine its unpacked copy in scratch (made at the end
  // of the solve; Im = 0)
  bool sol_packed = false;  // the last solve ran the packed real engine
  float2* sol_volume(int slot) { return sol_packed ? scratch : X[slot]; }

  int count_nnz(int slot, long long& total, std::vector<long long>* per_plane, cudaStream_t s) {
    const int nch = coo_chunks(P, std::max(nzl, 1));
    if (slot == counted_slot && nzl > 0) {  // the solution has not changed since the last count
      total = counted_total;
      if (per_plane) {
        const int cpp = nch / nzl;
        per_plane->assign(nzl, 0);
        for (int i = 0; i < nch; ++i) (*per_plane)[i / cpp] += h_counts[i];
      }
      return HOLO_OK;
    }
    HOLO_CUDA(dalloc(coo_counts, nch));
    HOLO_CUDA(dalloc(coo_offsets, nch));
    h_counts.resize(nch);
    h_offsets.resize(nch);
    if (nzl == 0) {
      total = 0;
      if (per_plane) per_plane->clear();
      return HOLO_OK;
    }
    HOLO_CUDA(coo_count(sol_volume(slot), P, nzl, coo_counts, s));
    HOLO_CUDA(cudaMemcpyAsync(h_counts.data(), coo_counts, sizeof(int) * nch, cudaMemcpyDeviceToHost, s));
    HOLO_CUDA(cudaStreamSynchronize(s));
    const int cpp = nch / nzl;
    long long run = 0;
    if (per_plane) per_plane->assign(nzl, 0);
    for (int i = 0; i < nch; ++i) {
      h_offsets[i] = run;
      run += h_counts[i];
      if (per_plane) (*per_plane)[i / cpp] += h_counts[i];
    }
    total = run;
    HOLO_CUDA(cudaMemcpyAsync(coo_offsets, h_offsets.data(), sizeof(long long) * nch, cudaMemcpyHostToDevice, s));
    counted_slot = slot;
    counted_total = run;
    return HOLO_OK;
  }

  // solver.py:254-379
  int solve(const double* b_dev, const holo_solver_config& cfg, holo_report& rep, cudaStream_t s) {
    nvtxRangePushA("holo_solve");
    struct PopOnExit {
      ~PopOnExit() { nvtxRangePop(); }
    } pop_on_exit;
    auto t0 = std::chrono::steady_clock::now();
    int rc;
    if (cfg.max_iters < 1) return fail(HOLO_ERR_INVALID, "max_iters must be >= 1");
    if (cfg.tv_inner_iters < 1) return fail(HOLO_ERR_INVALID, "tv_inner_iters must be >= 1");
    if (!(cfg.bt_shrink > 0.0 && cfg.bt_shrink < 1.0)) return fail(HOLO_ERR_INVALID, "bt_shrink must be in (0, 1)");
    if (cfg.lambda_l1 < 0 || cfg.lambda_tv < 0) return fail(HOLO_ERR_INVALID, "regularizer weights must be nonnegative");
    if (cfg.stop_tol < 0) return fail(HOLO_ERR_INVALID, "stop_tol must be nonnegative");
    if (cfg.step_policy != HOLO_POLICY_BACKTRACKING && cfg.step_policy != HOLO_POLICY_FIXED)
      return fail(HOLO_ERR_INVALID, "unknown step_policy");
    if (peer_broken)
      return fail(HOLO_ERR_NCCL, "an earlier peer spectrum reduction timed out: the rank group is out of step, "
                                 "recreate the handle");
    if ((rc = load_b(b_dev, s))) return rc;
    set_stack(cfg.real_nonnegative != 0);
    last = holo_report{};
    history.clear();
    have_solution = false;
    counted_slot = -1;
    const size_t vbytes = sizeof(float2) * (size_t)nzl * P;
    for (int i = 0; i < 3; ++i) {
      if (vbytes) HOLO_CUDA(cudaMemsetAsync(X[i], 0, vbytes, s));
      HOLO_CUDA(cudaMemsetAsync(S[i], 0, sizeof(float2) * P, s));
    }
    if ((rc = read_scalars(s))) return rc;
    const double f0 = h_scal[SC_F0];
    double step;
    if (cfg.step_size > 0) {
      step = cfg.step_size;
    } else if (cfg.real_nonnegative) {
      return fail(HOLO_ERR_INVALID, "real_nonnegative needs step_size (the reference's power-iteration estimate; "
                                    "see holo_power_iteration)");
    } else {
      const double sigma2 = (double)geom.nz;
      step = sigma2 > 0 ? 1.0 / (2.0 * sigma2) : 1.0;
    }
    int sx = 0, sxp = 0;  // x and x_prev both the zero volume (solver.py:289-290)
    double t = 1.0, last_obj = f0;
    int restarts = 0;
    bool diverged = false;
    for (int it = 0; it < cfg.max_iters; ++it) {
      double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
      const double beta = (t - 1.0) / tn;
      Attempt A{};
      if ((rc = iterate_from(sx, sxp, beta, step, cfg, A, s))) return rc;
      step = A.step;
      double obj = A.f_new + A.pen;
      int new_slot = A.slot;
      if (obj > last_obj && it > 0) {
        // adaptive restart (solver.py:339-349)
        restarts += 1;
        t = 1.0;
        tn = 1.0;
        if ((rc = iterate_from(sx, sx, 0.0, step, cfg, A, s))) return rc;
        step = A.step;
        obj = A.f_new + A.pen;
        new_slot = A.slot;
        if (obj > last_obj) {
          new_slot = sx;  // keep the previous iterate
          obj = last_obj;
        }
      }
      sxp = sx;
      sx = new_slot;
      t = tn;
      history.push_back(obj);
      if (obj > 1e6 * std::max(f0, 1e-300)) {
        diverged = true;
        break;
      }
      if (cfg.stop_tol > 0 && last_obj > 0) {
        if (std::fabs(last_obj - obj) / std::max(last_obj, 1e-300) < cfg.stop_tol) {
          last_obj = obj;
          break;
        }
      }
      last_obj = obj;
    }
    ix = sx;
    have_solution = true;
    sol_packed = packed;
    if (packed && nzl > 0) HOLO_CUDA(unpack_real(X[sx], scratch, nzl, P, s));
    long long nnz = 0;
    if ((rc = count_nnz(sx, nnz, nullptr, s))) return rc;
    if (nranks > 1) {
      double v = (double)nnz;
      HOLO_CUDA(cudaMemcpyAsync(scal, &v, sizeof(double), cudaMemcpyHostToDevice, s));
      if ((rc = allreduce_scalars(scal, 1, s))) return rc;
      if ((rc = read_scalars(s))) return rc;
      nnz = (long long)llround(h_scal[0]);
    }
    HOLO_CUDA(cudaStreamSynchronize(s));
    HOLO_CUDA(prof.harvest());
    const double V = (double)geom.nx * geom.ny * geom.nz;
    last.iterations = (int)history.size();
    last.restarts = restarts;
    last.diverged = diverged ? 1 : 0;
    last.step_size = step;
    last.final_sparsity = 1.0 - (double)nnz / V;
    last.f0 = f0;
    last.nnz = nnz;
    last.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rep = last;
    return diverged ? fail(HOLO_ERR_DIVERGED, "objective diverged at iteration " + std::to_string(history.size() - 1))
                    : HOLO_OK;
  }
};

}  // namespace holo

using holo::Engine;
using holo::fail;
using holo::g_err;

struct holo_handle {
  Engine e;
};

#define GUARD_HANDLE(h)                                                    \
  do {                                                                     \
    if (!(h)) return fail(HOLO_ERR_INVALID, "null handle");                \
    cudaError_t _se = cudaSetDevice((h)->e.device);                        \
    if (_se != cudaSuccess) return fail(HOLO_ERR_CUDA, cudaGetErrorString(_se)); \
  } while (0)

#define TRY(body)                                                          \
  try {                                                                    \
    body                                                                   \
  } catch (const std::exception& ex) {                                     \
    return fail(HOLO_ERR_CUDA, std::string("internal: ") + ex.what());    \
  } catch (...) {                                                          \
    return fail(HOLO_ERR_CUDA, "internal: unknown exception");            \
  }

extern "C" {

const char* holo_last_error(void) { return holo::g_err.c_str(); }
int holo_version(void) { return 1; }

int holo_debug_checks(uint32_t* bits) {
  cudaDeviceSynchronize();
  const unsigned v = holo::check_bits_kernels() | holo::check_bits_prox() | holo::check_bits_gfft();
  if (bits) *bits = v;
#ifdef HOLO_CHECKS
  return 1;
#else
  return 0;
#endif
}
int holo_shape_supported(int32_t nx, int32_t ny) { return holo::plan_supported(nx, ny) ? 1 : 0; }

int holo_create(const holo_geometry* geom, int device, holo_handle** out) {
  if (!geom || !out) return fail(HOLO_ERR_INVALID, "null argument");
  TRY({
    auto* h = new holo_handle();
    int rc = h->e.init(*geom, device, 0, 1);
    if (rc) {
      std::string keep = g_err;
      delete h;
      g_err = keep;
      return rc;
    }
    *out = h;
    return HOLO_OK;
  })
}

int holo_nccl_unique_id(void* out128) {
#ifdef HOLO_WITH_NCCL
  if (!out128) return fail(HOLO_ERR_INVALID, "null argument");
  if (!holo::nccl().ok) return fail(HOLO_ERR_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(HOLO_ERR_NCCL, ncclGetErrorString(r));
  std::memcpy(out128, &id, sizeof(id));
  return HOLO_OK;
#else
  (void)out128;
  return fail(HOLO_ERR_UNSUPPORTED, "built without NCCL");
#endif
}

int holo_create_sharded(const holo_geometry* geom, int device, const void* nccl_unique_id, int rank, int nranks,
                        holo_handle** out) {
  if (!geom || !out) return fail(HOLO_ERR_INVALID, "null argument");
  // one rank needs no communicator; HOLO_NCCL_SINGLE_RANK=1 keeps the NCCL path
  // anyway so the sharded plumbing can be exercised on a single GPU (tests)
  const char* force = std::getenv("HOLO_NCCL_SINGLE_RANK");
  if (nranks == 1 && !(force && force[0] == '1')) return holo_create(geom, device, out);
#ifdef HOLO_WITH_NCCL
  if (!nccl_unique_id) return fail(HOLO_ERR_INVALID, "null nccl id");
  if (!holo::nccl().ok) return fail(HOLO_ERR_NCCL, "libnccl.so.2 not loadable");
  TRY({
    auto* h = new holo_handle();
    int rc = h->e.init(*geom, device, rank, nranks);
    if (!rc) {
      ncclUniqueId id;
      std::memcpy(&id, nccl_unique_id, sizeof(id));
      ncclResult_t r = ncclCommInitRank(&h->e.comm, nranks, id, rank);
      if (r != ncclSuccess) rc = fail(HOLO_ERR_NCCL, ncclGetErrorString(r));
    }
    if (rc) {
      std::string keep = g_err;
      delete h;
      g_err = keep;
      return rc;
    }
    *out = h;
    return HOLO_OK;
  })
#else
  (void)device; (void)nccl_unique_id; (void)rank;
  return fail(HOLO_ERR_UNSUPPORTED, "built without NCCL");
#endif
}

int holo_create_local_group(const holo_geometry* geom, int device, int nranks, holo_handle** out) {
  if (!geom || !out) return fail(HOLO_ERR_INVALID, "null argument");
  if (nranks < 1 || nranks > holo::kMaxGroup) return fail(HOLO_ERR_INVALID, "nranks must be in [1, 8]");
  TRY({
    cudaError_t ce = cudaSetDevice(device);
    if (ce) return fail(HOLO_ERR_CUDA, cudaGetErrorString(ce));
    auto grp = std::make_shared<holo::LocalGroup>();
    ce = grp->init(nranks);
    if (ce) return fail(HOLO_ERR_CUDA, cudaGetErrorString(ce));
    for (int r = 0; r < nranks; ++r) out[r] = nullptr;
    for (int r = 0; r < nranks; ++r) {
      auto* h = new holo_handle();
      int rc = h->e.init(*geom, device, r, nranks);
      if (rc) {
        std::string keep = g_err;
        delete h;
        for (int q = 0; q < r; ++q) {
          delete out[q];
          out[q] = nullptr;
        }
        g_err = keep;
        return rc;
      }
      h->e.lgroup = grp;
      out[r] = h;
    }
    // the rank group reduces the forward spectrum through the peer kernels
    // (its members' buffers are plain pointers on this device)
    for (int r = 0; r < nranks && nranks > 1; ++r) {
      int rc = out[r]->e.ensure_peer_buffers();
      if (rc) return rc;
    }
    for (int r = 0; r < nranks && nranks > 1; ++r) {
      auto& e = out[r]->e;
      for (int j = 0; j < nranks; ++j) {
        e.pset.inbox[j] = out[j]->e.pr_inbox;
        e.pset.result[j] = out[j]->e.pr_result;
        e.pset.flags[j] = out[j]->e.pr_flags;
      }
      e.peer_on = true;
    }
    return HOLO_OK;
  })
}

int holo_peer_export(holo_handle* h, void* blob, int64_t* nbytes) {
  GUARD_HANDLE(h);
  if (!nbytes) return fail(HOLO_ERR_INVALID, "null argument");
  constexpr int64_t kBlob = 3 * (int64_t)sizeof(cudaIpcMemHandle_t) + 8;
  if (!blob) {
    *nbytes = kBlob;
    return HOLO_OK;
  }
  if (*nbytes < kBlob) return fail(HOLO_ERR_INVALID, "peer blob buffer too small");
  TRY({
    auto& e = h->e;
    if (e.nranks < 2 || e.nranks > holo::kMaxPeers) return fail(HOLO_ERR_INVALID, "peer reduction needs 2..8 ranks");
    if (int rc = e.ensure_peer_buffers()) return rc;
    cudaIpcMemHandle_t hd[3];
    HOLO_CUDA(cudaIpcGetMemHandle(&hd[0], e.pr_inbox));
    HOLO_CUDA(cudaIpcGetMemHandle(&hd[1], e.pr_result));
    HOLO_CUDA(cudaIpcGetMemHandle(&hd[2], e.pr_flags));
    std::memcpy(blob, hd, sizeof(hd));
    const int64_t L = e.pset.L;
    std::memcpy(static_cast<char*>(blob) + sizeof(hd), &L, 8);
    *nbytes = kBlob;
    return HOLO_OK;
  })
}

int holo_peer_import(holo_handle* h, const void* blobs, int64_t nbytes_each) {
  GUARD_HANDLE(h);
  if (!blobs) return fail(HOLO_ERR_INVALID, "null argument");
  TRY({
    auto& e = h->e;
    if (!e.pr_inbox) return fail(HOLO_ERR_INVALID, "holo_peer_export first");
    cudaIpcMemHandle_t hd[3];
    if (nbytes_each < (int64_t)sizeof(hd) + 8) return fail(HOLO_ERR_INVALID, "bad peer blob size");
    for (int j = 0; j < e.nranks; ++j) {
      if (j == e.rank) continue;
      const char* b = static_cast<const char*>(blobs) + (size_t)j * nbytes_each;
      int64_t L = 0;
      std::memcpy(hd, b, sizeof(hd));
      std::memcpy(&L, b + sizeof(hd), 8);
      if (L != e.pset.L) return fail(HOLO_ERR_INVALID, "peer slice length mismatch (different geometry?)");
      void* p[3];
      for (int k = 0; k < 3; ++k) {
        HOLO_CUDA(cudaIpcOpenMemHandle(&p[k], hd[k], cudaIpcMemLazyEnablePeerAccess));
        e.pr_mapped.push_back(p[k]);
      }
      e.pset.inbox[j] = static_cast<float2*>(p[0]);
      e.pset.result[j] = static_cast<float2*>(p[1]);
      e.pset.flags[j] = static_cast<unsigned long long*>(p[2]);
    }
    e.peer_on = true;
    return HOLO_OK;
  })
}

int64_t holo_peer_slice(int64_t plane_elems, int32_t nranks) {
  return nranks >= 1 ? holo::peer_slice(plane_elems, nranks) : 0;
}

int holo_destroy(holo_handle* h) {
  if (!h) return HOLO_OK;
  cudaSetDevice(h->e.device);
  delete h;
  return HOLO_OK;
}

int holo_local_planes(const holo_handle* h, int32_t* k_begin, int32_t* k_end) {
  if (!h || !k_begin || !k_end) return fail(HOLO_ERR_INVALID, "null argument");
  *k_begin = h->e.kb;
  *k_end = h->e.ke;
  return HOLO_OK;
}

int holo_operator_norm(holo_handle* h, int32_t real, double* sigma2) {
  GUARD_HANDLE(h);
  if (!sigma2) return fail(HOLO_ERR_INVALID, "null argument");
  if (!real) {
    *sigma2 = h->e.plan.any_propagating ? (double)h->e.geom.nz : 0.0;
    return HOLO_OK;
  }
  TRY({ return h->e.real_opnorm_value(*sigma2, h->e.stream); })
}

int holo_solve_device(holo_handle* h, const double* b_dev, const holo_solver_config* cfg, holo_report* rep,
                      void* stream) {
  GUARD_HANDLE(h);
  if (!b_dev || !cfg || !rep) return fail(HOLO_ERR_INVALID, "null argument");
  TRY({ return h->e.solve(b_dev, *cfg, *rep, h->e.st(stream)); })
}

int holo_solve(holo_handle* h, const double* b_host, const holo_solver_config* cfg, holo_report* rep) {
  GUARD_HANDLE(h);
  if (!b_host || !cfg || !rep) return fail(HOLO_ERR_INVALID, "null argument");
  TRY({
    Engine& e = h->e;
    int rc = e.ensure_planes();
    if (rc) return rc;
    HOLO_CUDA(cudaMemcpyAsync(e.b64, b_host, sizeof(double) * e.P, cudaMemcpyHostToDevice, e.stream));
    return e.solve(e.b64, *cfg, *rep, e.stream);
  })
}

int holo_history(const holo_handle* h, double* out, int32_t cap, int32_t* n) {
  if (!h || !n) return fail(HOLO_ERR_INVALID, "null argument");
  const auto& hist = h->e.history;
  *n = (int32_t)hist.size();
  if (out) std::memcpy(out, hist.data(), sizeof(double) * std::min<size_t>(hist.size(), (size_t)std::max(cap, 0)));
  return HOLO_OK;
}

int holo_plane_nnz(holo_handle* h, int64_t* nnz_per_local_plane) {
  GUARD_HANDLE(h);
  if (!nnz_per_local_plane) return fail(HOLO_ERR_INVALID, "null argument");
  if (!h->e.have_solution) return fail(HOLO_ERR_INVALID, "no solution: call holo_solve first");
  TRY({
    long long tot = 0;
    std::vector<long long> per;
    int rc = h->e.count_nnz(h->e.ix, tot, &per, h->e.stream);
    if (rc) return rc;
    HOLO_CUDA(cudaStreamSynchronize(h->e.stream));
    for (size_t i = 0; i < per.size(); ++i) nnz_per_local_plane[i] = per[i];
    return HOLO_OK;
  })
}

// memcpy split over host threads (the destination is fresh pageable memory:
// the copy also takes its first-touch page faults, which parallelise)
static void par_memcpy(char* dst, const char* src, size_t n) {
  static const int nt = (int)std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
  if (nt <= 1 || n < (size_t)(4u << 20)) {
    std::memcpy(dst, src, n);
    return;
  }
  std::vector<std::thread> pool;
  const size_t part = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const size_t o = (size_t)t * part;
    if (o >= n) break;
    pool.emplace_back([=] { std::memcpy(dst + o, src + o, std::min(part, n - o)); });
  }
  for (auto& th : pool) th.join();
}

// Device -> pageable host through a pinned double buffer: the DMA of chunk
// i+1 overlaps the threaded copy-out of chunk i (pageable cudaMemcpy runs at a
// few GB/s; this path is bounded by the host copy-out).
static int d2h_staged(Engine& e, void* dst, const void* src, size_t n, cudaStream_t s) {
  constexpr size_t kChunk = 32u << 20;
  for (int i = 0; i < 2; ++i) {
    if (!e.stage_host[i]) HOLO_CUDA(cudaHostAlloc(&e.stage_host[i], kChunk, cudaHostAllocDefault));
    if (!e.stage_ev[i]) HOLO_CUDA(cudaEventCreateWithFlags(&e.stage_ev[i], cudaEventDisableTiming));
  }
  const size_t nchunk = (n + kChunk - 1) / kChunk;
  auto issue = [&](size_t c) -> cudaError_t {
    const size_t o = c * kChunk, len = std::min(kChunk, n - o);
    cudaError_t err = cudaMemcpyAsync(e.stage_host[c & 1], (const char*)src + o, len, cudaMemcpyDeviceToHost, s);
    return err ? err : cudaEventRecord(e.stage_ev[c & 1], s);
  };
  for (size_t c = 0; c < std::min<size_t>(2, nchunk); ++c) HOLO_CUDA(issue(c));
  for (size_t c = 0; c < nchunk; ++c) {
    HOLO_CUDA(cudaEventSynchronize(e.stage_ev[c & 1]));
    const size_t o = c * kChunk, len = std::min(kChunk, n - o);
    par_memcpy((char*)dst + o, (const char*)e.stage_host[c & 1], len);
    if (c + 2 < nchunk) HOLO_CUDA(issue(c + 2));
  }
  return HOLO_OK;
}

static int export_coo(holo_handle* h, int32_t* rows, int32_t* cols, void* vals, int64_t cap, int64_t* nnz, bool host,
                      cudaStream_t s) {
  Engine& e = h->e;
  if (!e.have_solution) return fail(HOLO_ERR_INVALID, "no solution: call holo_solve first");
  long long tot = 0;
  int rc = e.count_nnz(e.ix, tot, nullptr, s);
  if (rc) return rc;
  if (nnz) *nnz = tot;
  if (tot > cap) return fail(HOLO_ERR_INVALID, "COO capacity too small");
  if (tot == 0) return HOLO_OK;
  if (!host) {
    HOLO_CUDA(holo::coo_compact(e.sol_volume(e.ix), e.P, e.geom.nx, e.nzl, e.coo_offsets, rows, cols, (float2*)vals,
                                nullptr, s));
    return HOLO_OK;
  }
  if (tot > e.coo_cap) {  // grow-only device staging, reused across exports
    cudaFree(e.coo_rows);
    cudaFree(e.coo_cols);
    cudaFree(e.coo_vals);
    e.coo_rows = e.coo_cols = nullptr;
    e.coo_vals = nullptr;
    const long long cap2 = tot + tot / 4;
    HOLO_CUDA(cudaMalloc(&e.coo_rows, sizeof(int32_t) * cap2));
    HOLO_CUDA(cudaMalloc(&e.coo_cols, sizeof(int32_t) * cap2));
    HOLO_CUDA(cudaMalloc(&e.coo_vals, sizeof(double2) * cap2));
    e.coo_cap = cap2;
  }
  // values widened to complex128 on the device: the caller's arrays are final
  HOLO_CUDA(holo::coo_compact(e.sol_volume(e.ix), e.P, e.geom.nx, e.nzl, e.coo_offsets, e.coo_rows, e.coo_cols, nullptr,
                              e.coo_vals, s));
  if ((rc = d2h_staged(e, rows, e.coo_rows, sizeof(int32_t) * tot, s))) return rc;
  if ((rc = d2h_staged(e, cols, e.coo_cols, sizeof(int32_t) * tot, s))) return rc;
  return d2h_staged(e, vals, e.coo_vals, sizeof(double2) * tot, s);
}

int holo_export_coo_host(holo_handle* h, int32_t* rows, int32_t* cols, double* vals, int64_t cap, int64_t* nnz) {
  GUARD_HANDLE(h);
  TRY({ return export_coo(h, rows, cols, vals, cap, nnz, true, h->e.stream); })
}

int holo_export_coo_device(holo_handle* h, int32_t* rows, int32_t* cols, float* vals, int64_t cap, int64_t* nnz,
                           void* stream) {
  GUARD_HANDLE(h);
  TRY({ return export_coo(h, rows, cols, vals, cap, nnz, false, h->e.st(stream)); })
}

int holo_solution_device(holo_handle* h, void** x) {
  if (!h || !x) return fail(HOLO_ERR_INVALID, "null argument");
  if (!h->e.have_solution) return fail(HOLO_ERR_INVALID, "no solution: call holo_solve first");
  *x = h->e.sol_volume(h->e.ix);
  return HOLO_OK;
}

int holo_op_transfer(holo_handle* h, int32_t k0, int32_t k1, int32_t conj, void* out, void* stream) {
  GUARD_HANDLE(h);
  if (!out || k0 < 0 || k1 < k0) return fail(HOLO_ERR_INVALID, "bad plane range");
  if (k1 == k0) return HOLO_OK;
  HOLO_CUDA(holo::transfer_stack(h->e.plan, k0, k1, conj != 0, (float2*)out, h->e.st(stream)));
  return HOLO_OK;
}

int holo_op_fft2(holo_handle* h, void* data, int32_t nplanes, int32_t inverse, void* stream) {
  GUARD_HANDLE(h);
  if (!data || nplanes < 0) return fail(HOLO_ERR_INVALID, "bad argument");
  if (nplanes == 0) return HOLO_OK;
  Engine& e = h->e;
  cudaStream_t s = e.st(stream);
  float2* d = (float2*)data;
  const float sc = inverse ? 1.0f / (float)e.P : 1.0f;
  HOLO_CUDA(holo::fft_rows(e.plan, d, d, (long long)nplanes * e.geom.ny, inverse != 0, 1.0f, s));
  HOLO_CUDA(holo::fft_cols(e.plan, d, d, nplanes, inverse != 0, sc, s));
  return HOLO_OK;
}

int holo_op_forward(holo_handle* h, const void* x, void* out, void* stream) {
  GUARD_HANDLE(h);
  if (!x || !out) return fail(HOLO_ERR_INVALID, "null argument");
  TRY({
    Engine& e = h->e;
    cudaStream_t s = e.st(stream);
    int rc = e.ensure_scratch();
    if (rc) return rc;
    e.set_stack(false);  // one complex plane per local plane
    if (e.sol_packed) e.have_solution = false;  // (its unpacked copy lives in scratch, overwritten here)
    if ((rc = e.forward_spectrum((const float2*)x, e.S[0], s))) return rc;
    HOLO_CUDA(holo::apply_mask(e.plan, e.S[0], 1, s));
    HOLO_CUDA(holo::fft_rows(e.plan, e.S[0], e.R, e.geom.ny, true, 1.0f, s));
    HOLO_CUDA(holo::fft_cols(e.plan, e.R, e.R, 1, true, 1.0f / (float)e.P, s));
    HOLO_CUDA(holo::real_part(e.R, (float*)out, e.P, 1.0f, s));
    return HOLO_OK;
  })
}

int holo_op_adjoint(holo_handle* h, const void* r, void* out, double scale, void* stream) {
  GUARD_HANDLE(h);
  if (!r || !out) return fail(HOLO_ERR_INVALID, "null argument");
  TRY({
    Engine& e = h->e;
    cudaStream_t s = e.st(stream);
    int rc = e.ensure_planes();
    if (rc) return rc;
    HOLO_CUDA(holo::real_to_complex((const float*)r, e.R, e.P, s));
    HOLO_CUDA(holo::fft_rows(e.plan, e.R, e.R, e.geom.ny, false, 1.0f, s));
    HOLO_CUDA(holo::fft_cols(e.plan, e.R, e.R, 1, false, 1.0f, s));
    HOLO_CUDA(holo::apply_mask(e.plan, e.R, 1, s));
    HOLO_CUDA(holo::adj_cols(e.plan, e.R, (float2*)out, e.nzl, e.kb, s));
    HOLO_CUDA(holo::fft_rows(e.plan, (float2*)out, (float2*)out, (long long)e.nzl * e.geom.ny, true,
                             (float)(scale / (double)e.P), s));
    return HOLO_OK;
  })
}

int holo_op_prox_fl(holo_handle* h, const void* v, void* out, int32_t nplanes, int32_t ny, int32_t nx, double tau_l1,
                    double tau_tv, int32_t inner, void* stream) {
  GUARD_HANDLE(h);
  if (!v || !out || nplanes < 0 || ny < 1 || nx < 1 || ny > 65535 || nx > 65535)
    return fail(HOLO_ERR_INVALID, "bad argument");
  if (tau_l1 < 0 || tau_tv < 0) return fail(HOLO_ERR_INVALID, "tau must be nonnegative");
  if (inner < 1) return fail(HOLO_ERR_INVALID, "inner_iters must be >= 1");
  if (nplanes == 0) return HOLO_OK;
  TRY({
    Engine& e = h->e;
    cudaStream_t s = e.st(stream);
    holo::ProxArgs a;
    int rc = e.ensure_prox(a, nplanes, ny, nx, inner, s);
    if (rc) return rc;
    uint8_t* force = nullptr;
    double* pout = nullptr;
    int* nf = nullptr;
    double* sc = nullptr;
    HOLO_CUDA(cudaMallocAsync(&force, nplanes, s));
    HOLO_CUDA(cudaMallocAsync(&pout, sizeof(double) * 4 * nplanes, s));
    HOLO_CUDA(cudaMallocAsync(&nf, sizeof(int) * nplanes, s));
    HOLO_CUDA(cudaMallocAsync(&sc, sizeof(double) * 8, s));
    HOLO_CUDA(cudaMemsetAsync(force, 0, nplanes, s));
    a.x = (const float2*)v;
    a.xnew = (float2*)out;
    a.tau_l1 = (float)tau_l1;
    a.tau_tv = (float)tau_tv;
    a.lr_tv = tau_tv > 0 ? (float)(1.0 / (8.0 * tau_tv)) : 0.f;
    double fails = 0;
    for (int round = 0; round < 3; ++round) {
      holo::ProxArgs f = a;
      if (round > 0) f.force = force;
      HOLO_CUDA(holo::prox(f, s));
      HOLO_CUDA(holo::prox_reduce(f, tau_tv, tau_tv > 0, force, pout, nf, s));
      HOLO_CUDA(holo::plane_total(pout, nf, nplanes, sc, s));
      HOLO_CUDA(cudaMemcpyAsync(&fails, sc + 4, sizeof(double), cudaMemcpyDeviceToHost, s));
      HOLO_CUDA(cudaStreamSynchronize(s));
      if (fails < 0.5) break;
    }
    cudaFreeAsync(force, s);
    cudaFreeAsync(pout, s);
    cudaFreeAsync(nf, s);
    cudaFreeAsync(sc, s);
    return HOLO_OK;
  })
}

int holo_profile_enable(holo_handle* h, int32_t on) {
  if (!h) return fail(HOLO_ERR_INVALID, "null handle");
  h->e.prof.on = on != 0;
  h->e.prof.reset();
  return HOLO_OK;
}

int holo_profile_classes(holo_handle* h, uint32_t mask) {
  if (!h) return fail(HOLO_ERR_INVALID, "null handle");
  h->e.prof.mask = mask;
  return HOLO_OK;
}

int holo_profile_read(holo_handle* h, int32_t* n, char* names, double* ms, int64_t* counts) {
  if (!h || !n) return fail(HOLO_ERR_INVALID, "null argument");
  *n = holo::PK_N;
  for (int i = 0; i < holo::PK_N; ++i) {
    if (names) {
      std::memset(names + 32 * i, 0, 32);
      std::strncpy(names + 32 * i, holo::kProfNames[i], 31);
    }
    if (ms) ms[i] = h->e.prof.ms[i];
    if (counts) counts[i] = h->e.prof.cnt[i];
  }
  return HOLO_OK;
}

int64_t holo_launch_count(void) { return holo::launch_count(); }

int holo_power_iteration(holo_handle* h, const void* v0, int32_t iters, int32_t real, double* sigma2, void* stream) {
  GUARD_HANDLE(h);
  if (!v0 || !sigma2 || iters < 1) return fail(HOLO_ERR_INVALID, "bad argument");
  TRY({ return h->e.power_iteration((const float2*)v0, iters, real != 0, *sigma2, h->e.st(stream)); })
}

}  // extern "C"
