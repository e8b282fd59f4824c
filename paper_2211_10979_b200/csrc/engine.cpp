// engine.cpp — libsimplex host engine and C ABI (include/libsimplex.h).
//
// One handle = one process's share of the tableau on one GPU:
//   * column partition of the n+m non-rhs columns into P contiguous slabs of width
//     floor((n+m)/P) or +1, remainder to the lowest parts, rhs replicated
//     on every part;
//   * P = nranks (one process per GPU, NCCL over NVLink) or virtual_ranks (several
//     slabs on one GPU exchanging through device memory: same kernels, same data
//     flow, used to test the multi-GPU path on one GPU);
//   * the per-pivot loop runs entirely on the device inside
//     captured CUDA-graph segments of S pivots; the host only looks at the status
//     word once per segment, with two segments in flight so the GPU never waits.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/libsimplex.h"
#include "device.cuh"
#include "host_lane.h"
#include "kernels.h"

namespace {

thread_local std::string g_err;

simplex_err fail(simplex_err code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) return fail(e_ == cudaErrorMemoryAllocation ? SIMPLEX_E_OOM : SIMPLEX_E_CUDA, \
                                       std::string(#x) + ": " + cudaGetErrorString(e_));        \
  } while (0)

#define NK(x)                                                                                   \
  do {                                                                                          \
    ncclResult_t r_ = (x);                                                                      \
    if (r_ != ncclSuccess) return fail(SIMPLEX_E_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

#define RET(x)                                    \
  do {                                            \
    simplex_err e_ = (x);                         \
    if (e_ != SIMPLEX_OK) return e_;              \
  } while (0)

long long roundup(long long a, long long b) { return (a + b - 1) / b * b; }
constexpr int kMaxPeersHost = sx::kMaxPeers;

struct Slab {
  sx::SlabView v{};
  int q = 1;             // k_update: rows swept concurrently (threads / (ld/2))
  int upd_grid = 1;
  int sel_grid = 1;
  int look_grid = 0;     // look-ahead selection: CTAs of its single thread-block cluster
  int nc = 0, cw = 0, Gr = 0;   // rank-s pass: column chunks, chunk width, row groups
  double* T2 = nullptr;          // second tableau buffer of the look-ahead software pipeline
};

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    if (prev_ != dev) cudaSetDevice(dev);
    dev_ = dev;
  }
  ~DeviceGuard() {
    if (prev_ != dev_) cudaSetDevice(prev_);
  }

 private:
  int prev_ = 0, dev_ = 0;
};

}  // namespace

struct simplex_s {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;       // internal non-blocking stream (graphs are captured here)
  cudaStream_t user_stream = nullptr;  // caller's stream (NULL = legacy default stream)
  cudaEvent_t ev_user = nullptr, ev_loop0 = nullptr, ev_loop1 = nullptr;
  cudaEvent_t ev_done[2] = {nullptr, nullptr};
  long long m = 0, n = 0, W = 0, arts = 0;   // arts: artificial columns (rows with b_i < 0)
  std::vector<int> art_rows;               // rows with b_i < 0 at create (1-based)
  int nranks = 1, rank = 0, nslabs = 1, nparts = 1;
  simplex_options opt{};
  long long cap = 0;
  std::vector<Slab> slabs;
  std::vector<void*> allocs;
  // exchange
  ncclComm_t comm = nullptr;
  double* send = nullptr;
  double* recv = nullptr;
  long long xstride = 0;
  bool p2p = false;                     // multi-part look-ahead exchanges over peer memory (no NCCL)
  bool mblock = false;                  // ... with the whole block's selection in one k_mblock launch
  bool mpipe = false;                   // ... and that selection overlapped with the previous block's
                                        //     slab passes (two tableau buffers per slab, §8)
  std::vector<cudaStream_t> xs;         // virtual slabs under k_mblock: one stream each (co-resident)
  cudaEvent_t ev_fork = nullptr;
  std::vector<cudaEvent_t> ev_join;
  unsigned long long* xll = nullptr;    // peer-memory gather buffer (LL words, device.cuh XPeers)
  std::vector<void*> ipc_open;          // peer allocations mapped with cudaIpcOpenMemHandle
  std::vector<sx::XPeers> xpeers;       // per slab
  // extraction scratch
  double* d_x = nullptr;
  double* d_y = nullptr;
  double* d_obj = nullptr;
  double* d_b = nullptr;
  double* d_res = nullptr;              // simplex_solve_lp: {objective, status, pivots, error bits}
  double* h_res = nullptr;              // pinned copy of it
  double* d_stage = nullptr;            // simplex_solve_lp with host inputs: A, b, c staged on the device
  unsigned long long* d_hash = nullptr;
  double* d_fcol = nullptr;             // Phase I drive-out: staged [flag, pivot column] per rank
  long long* d_fj = nullptr;            // ... each part's first eligible column, then the minimum
  sx::DevState* h_state = nullptr;  // pinned, 3 slots: 2 segment mirrors + 1 sync copy
  unsigned int* h_err = nullptr;    // pinned, one error word per slab (load)
  // graph segments
  int S = 32;                       // pivots per captured graph segment
  int look = 1;                     // pivots per tableau pass (>1: rank-s look-ahead)
  bool overlap = false;             // look-ahead software pipeline: select block b+1 during pass b
  bool look_cache = true;           // pipelined selection keeps the previous bank in shared memory
  int pass_cfg = 0;                 // k_update_s configuration (kernels.cu kPassCfgs)
  bool pdl = true;                  // programmatic dependent launch between pivot kernels
  bool force_nccl = false;          // exchange = 1 on one part: 1-rank NCCL exchange on one GPU
  bool small = false;               // the whole solve in one k_solve_small launch (tableau in smem)
  // hybrid CPU lane (options.host_share > 0): the host owns the last columns
  bool hybrid = false;
  sx::HostLane lane;
  double* h_slot = nullptr;         // pinned: the GPU part's candidate slot [v, k bits, col[0..m]]
  double* h_wcol = nullptr;         // pinned: the winning column when the host lane wins
  double* d_wcol = nullptr;         // ... its device copy (k_force stages it)
  cudaEvent_t ev_slot = nullptr;
  bool slot_ready = false;          // k_pack + D2H of the GPU candidate enqueued for the next pivot
  std::vector<double> wcol;         // the winning column (host copy) of the current pivot
  double host_ms = 0.0, host_wait_ms = 0.0;
  bool graphs_ready = false;
  cudaGraphExec_t seg[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> tev[2];
  // host view of the loop
  int status = SIMPLEX_RUNNING;
  bool faulted = false;             // latched after an exchange timeout or a CUDA/NCCL error in
                                    // the loop: every later call except destroy -> E_STATE
  int phase = 2;                    // 1 while the Phase I objective is being optimized
  bool drive_pending = false;       // Phase I ended; its drive-out of artificials not finished yet
  std::vector<int> drive_rows;      // rows whose basic variable was artificial when Phase I ended
  long long drive_done = 0;         // listed rows handled (DevState.drive_next)
  long long xcol_stride() const { return roundup(m + 2, 2); }
  long long it = 0;
  // stats
  long long graph_launches = 0, kernel_launches = 0, upd_launches = 0;
  double upd_ms = 0.0, loop_ms = 0.0;

  template <class T>
  simplex_err dalloc(T** p, size_t count) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
    if (e != cudaSuccess)
      return fail(SIMPLEX_E_OOM, std::string("cudaMalloc(") + std::to_string(count * sizeof(T)) +
                                     " B): " + cudaGetErrorString(e));
    allocs.push_back(q);
    *p = static_cast<T*>(q);
    return SIMPLEX_OK;
  }

  sx::XView xview() const {
    sx::XView x{};
    x.nparts = nparts;
    x.recv = gathered() ? recv : nullptr;
    x.stride = xstride;
    return x;
  }

  // the entering column travels through the exchange buffer (pack -> gather -> select)
  bool gathered() const { return nparts > 1 || force_nccl; }
  bool use_nccl() const { return nranks > 1 || force_nccl; }
  int kernels_per_pivot() const { return nslabs * (2 + (gathered() ? 1 : 0)); }
  // graph steps per segment; the pipeline alternates two tableau buffers, so an even count
  // brings the tableau back to buffer 0 at every segment boundary
  bool time_pass() const {                     // the pipelined pass is timed on the device
    static const bool time_sel = sx::experiment_env("SIMPLEX_TIME_SELECT") != nullptr;
    return opt.time_kernels && (overlap || mpipe) && !time_sel;
  }
  int steps_per_segment() const {
    if (look == 1) return S;
    const int q = std::max(1, S / look);
    return (overlap || mpipe) ? (q + 1) / 2 * 2 : q;
  }
  int kernels_per_segment() const {
    if (look == 1) return S * kernels_per_pivot();
    if (gathered()) return steps_per_segment() * nslabs * (mblock ? 2 : look + 2);   // selection, pass
    return (look > sx::kMaxLook ? 3 : 2) * steps_per_segment();
  }

  simplex_err enter() {
    // order our stream after whatever the caller queued on its stream (e.g. inputs)
    CK(cudaEventRecord(ev_user, user_stream));
    CK(cudaStreamWaitEvent(stream, ev_user, 0));
    return SIMPLEX_OK;
  }

  simplex_err setup(long long m_, long long n_, const double* b, const simplex_options* o);
  simplex_err scan_b(const double* b, std::vector<int>* art_of_row, std::vector<int>* neg);
  simplex_err phase_transition();
  simplex_err load(const double* A, const double* b, const double* c, bool first);
  simplex_err build_graphs();
  simplex_err enqueue_pivot(int slot, int t);
  simplex_err run(long long max_pivots, long long* done);
  simplex_err run_small(long long max_pivots, long long* done);
  simplex_err solve_lp_small(const double* A, const double* b, const double* c, double* x, double* y,
                             double* objective, long long* pivots);
  simplex_err run_hybrid(long long max_pivots, long long* done);
  simplex_err load_lane(const double* A, const double* b, const double* c);
  simplex_err enqueue_gpu_candidate();
  simplex_err flush_all();
  void release();
  simplex_err setup_p2p();
  // the multi-part selection of one block: one k_mblock per slab (forked onto the selection
  // streams when there are several slabs or the passes run concurrently); join = false leaves the
  // join to the caller (after the concurrent passes)
  simplex_err mselect(int q, int bown, int bpre, bool join) {
    if (xs.empty()) {
      const Slab& sl = slabs[0];
      CK(sx::launch_mblock(sl.v, q ? sl.T2 : sl.v.T, nparts, xstride, look, bown, bpre, opt.tol_opt, opt.tol_piv,
                           sl.look_grid, xpeers[0], stream));
      return SIMPLEX_OK;
    }
    CK(cudaEventRecord(ev_fork, stream));
    for (int sidx = 0; sidx < nslabs; ++sidx) {
      const Slab& sl = slabs[sidx];
      cudaStream_t x = xs[(size_t)sidx];
      CK(cudaStreamWaitEvent(x, ev_fork, 0));
      CK(sx::launch_mblock(sl.v, q ? sl.T2 : sl.v.T, nparts, xstride, look, bown, bpre, opt.tol_opt, opt.tol_piv,
                           sl.look_grid, xpeers[(size_t)sidx], x));
      CK(cudaEventRecord(ev_join[(size_t)sidx], x));
    }
    if (join) RET(mjoin());
    return SIMPLEX_OK;
  }
  simplex_err mjoin() {
    for (auto e : ev_join) CK(cudaStreamWaitEvent(stream, e, 0));
    return SIMPLEX_OK;
  }
};

// Rows with b_i < 0 (1-based, ascending) and their artificial index (reading p1).
simplex_err simplex_s::scan_b(const double* b, std::vector<int>* art_of_row, std::vector<int>* neg) {
  std::vector<double> hb((size_t)m);
  // ordered after the caller's stream: every caller runs enter() first
  CK(cudaMemcpyAsync(hb.data(), b, sizeof(double) * m, cudaMemcpyDefault, stream));
  CK(cudaStreamSynchronize(stream));
  art_of_row->assign((size_t)m, -1);
  neg->clear();
  for (long long i = 0; i < m; ++i)
    if (hb[i] < 0.0) {
      (*art_of_row)[i] = (int)neg->size();
      neg->push_back((int)(i + 1));
    }
  return SIMPLEX_OK;
}

simplex_err simplex_s::setup(long long m_, long long n_, const double* b, const simplex_options* o) {
  m = m_;
  n = n_;
  opt = *o;
  nranks = std::max(1, opt.nranks);
  rank = opt.rank;
  nslabs = std::max(1, opt.virtual_ranks);
  if (rank < 0 || rank >= nranks) return fail(SIMPLEX_E_ARG, "rank out of range");
  if (nslabs > 1 && nranks > 1) return fail(SIMPLEX_E_ARG, "virtual_ranks requires nranks == 1");
  nparts = nranks * nslabs;
  if (nparts > n + m) return fail(SIMPLEX_E_ARG, "more column parts than columns");
  if (m + 1 > INT_MAX / 2 || n + m > INT_MAX / 2) return fail(SIMPLEX_E_ARG, "dimensions too large");
  cap = opt.max_pivots > 0 ? opt.max_pivots : 20 * (m + n);
  S = opt.segment_pivots > 0 ? opt.segment_pivots : 32;
  if (const char* e = sx::experiment_env("SIMPLEX_NO_PDL")) pdl = !(e[0] == '1');
  if (const char* e = sx::experiment_env("SIMPLEX_NO_LOOK_CACHE")) look_cache = !(e[0] == '1');
  // exchange = 1 on ONE column part: gather the candidate columns through a 1-rank NCCL
  // communicator (the multi-GPU data flow, NCCL flavour, testable on one GPU)
  force_nccl = opt.exchange == 1 && nranks == 1 && nslabs == 1;
  // 0 = automatic: rank-16 look-ahead on one column part, one pivot per pass otherwise
  // 0 = automatic: rank-16 look-ahead (one part: pipelined with the pass; several parts: one
  // exchange of candidate columns per selected pivot, then one pass per block)
  look = opt.lookahead > 0 ? opt.lookahead : sx::kMaxLook;
  if (look > sx::kColS) return fail(SIMPLEX_E_ARG, "lookahead larger than 32");
  if (look > sx::kMaxLook && nparts > 1)
    return fail(SIMPLEX_E_ARG, "lookahead 17..32 (pair schedule) runs on one column part only");
  // 17..32: the pair schedule — two selections (bank 0, then bank 1 chaining bank 0) and ONE
  // pass applying both banks; select-then-pass (no pipeline)
  overlap = look > 1 && look <= sx::kMaxLook && opt.overlap != 0 && nparts == 1 && !force_nccl;
  if (opt.exchange < 0 || opt.exchange > 3) return fail(SIMPLEX_E_ARG, "exchange must be 0, 1, 2 or 3");
  // multi-part look-ahead on several ranks: peer-memory exchange unless NCCL is asked for
  // (peer reachability is checked once the device is known); the 1-rank NCCL hook keeps NCCL
  // (one GPU, virtual slabs: only when asked for — there the protocol is pure overhead, the
  // stream already orders the parts; measured +6 us per k_mlook launch for the system fence)
  p2p = look > 1 && nparts > 1 && !force_nccl && (opt.exchange >= 2 || (opt.exchange == 0 && nranks > 1));
  if (p2p && nranks > kMaxPeersHost) return fail(SIMPLEX_E_ARG, "peer-memory exchange supports up to 8 ranks");

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(SIMPLEX_E_CUDA, "no CUDA device (libsimplex has no CPU fallback)");
  if (opt.device >= 0) {
    if (opt.device >= ndev) return fail(SIMPLEX_E_ARG, "device ordinal out of range");
    device = opt.device;
  } else {
    CK(cudaGetDevice(&device));
  }
  CK(cudaSetDevice(device));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  user_stream = static_cast<cudaStream_t>(opt.stream);
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ev_user, cudaEventDisableTiming));
  RET(enter());                     // b may have been written on the caller's stream
  // Phase I (NEXT #2): one artificial column per row with b_i < 0
  std::vector<int> art_of_row;
  RET(scan_b(b, &art_of_row, &art_rows));
  arts = (long long)art_rows.size();
  W = n + m + arts + 1;
  if (arts > 0 && !opt.phase1) return fail(SIMPLEX_E_NEG_RHS, "b has a negative entry and phase1 = 0");
  // lookahead = 0 (automatic) on a tableau that fits in one CTA's shared memory, one column part,
  // no Phase I: the latency path — the whole solve in ONE k_solve_small launch
  hybrid = opt.host_share > 0.0;
  if (hybrid) {
    if (!(opt.host_share < 1.0)) return fail(SIMPLEX_E_ARG, "host_share must be in [0, 1)");
    if (nparts != 1) return fail(SIMPLEX_E_ARG, "host_share needs one GPU rank and no virtual ranks");
    if (opt.lookahead > 1) return fail(SIMPLEX_E_ARG, "host_share needs lookahead 0 or 1 (one pivot per pass)");
    if (arts > 0) return fail(SIMPLEX_E_ARG, "host_share needs b >= 0 (no Phase I)");
    if (force_nccl) return fail(SIMPLEX_E_ARG, "host_share excludes exchange = 1");
    lane.m = m;
    lane.n = n;
    lane.W = n + m + 1;
    lane.hw = std::min<long long>(n + m - 1, std::max<long long>(1, std::llround(opt.host_share * (double)(n + m))));
    lane.c0 = n + m - lane.hw;
    lane.rule = opt.pivot_rule;
    lane.threads = opt.host_threads;
    look = 1;
    overlap = false;
  }
  small = !hybrid && opt.lookahead == 0 && nparts == 1 && arts == 0 && !force_nccl &&
          sx::small_smem_bytes((int)(m + 1), (int)(n + m)) <= sx::small_smem_max();
  if (small) {
    look = 1;
    overlap = false;
  }
  if (overlap) {
    // the pipeline needs a second tableau buffer: fall back to select-then-pass in place when
    // two tableaux (+10 %) do not fit in the free device memory
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const double tab = 8.0 * (double)(m + 1) * (double)roundup(W, 16);
    if (2.2 * tab > (double)free_b) overlap = false;
  }

  CK(cudaEventCreate(&ev_loop0));
  CK(cudaEventCreate(&ev_loop1));
  for (auto& e : ev_done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&h_state), 3 * sizeof(sx::DevState), cudaHostAllocDefault));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&h_err), sizeof(unsigned int) * std::max(1, nslabs), cudaHostAllocDefault));

  // ---- column partition: part p = rank * nslabs + s
  slabs.resize(nslabs);
  for (int s = 0; s < nslabs; ++s) {
    const long long p = (long long)rank * nslabs + s;
    Slab& sl = slabs[s];
    sx::SlabView& v = sl.v;
    int64_t c0 = 0, w = 0;
    RET(simplex_partition(n + m + arts, nparts, p, &c0, &w));
    if (hybrid) w = lane.c0;                     // the GPU keeps columns [0, c0 of the host lane)
    v.c0 = c0;
    v.w = (int)w;
    v.rows = (int)(m + 1);
    v.rule = opt.pivot_rule;
    v.arts = (int)arts;
    v.ld = roundup(v.w + 1, 16);
    v.nslot = (int)((v.ld / 2 + 31) / 32);
    sl.sel_grid = (int)std::min<long long>((v.rows + sx::kThreads - 1) / sx::kThreads, 2LL * sms);
    if (look > 1) {
      sl.look_grid = sx::lookahead_cluster_size();
      if (sl.look_grid < 1) return fail(SIMPLEX_E_CUDA, "look-ahead selection cluster cannot be scheduled");
      if (s == 0 && p2p) {
        // one k_mblock per part and block when every part's cluster can be resident at once (a
        // rank per GPU; virtual slabs: nslabs clusters on this GPU, each on its own stream), else
        // one k_mlook per pivot (also SIMPLEX_NO_MBLOCK=1, experiment hook); pipelined with the
        // slab passes (overlap = 1) when two tableau buffers per slab fit
        mblock = opt.exchange != 3 && sx::mblock_max_clusters(sl.look_grid, v.rows) >= nslabs;
        if (mblock && opt.overlap != 0) {
          // pipelined whenever two buffers per slab fit; with SEVERAL slabs on this GPU (virtual
          // ranks) only up to 2.5 GB of slab stream per block: beyond it the one-GPU emulation, where
          // the P passes share one HBM, measured the selections starved by the concurrent passes
          // (DESIGN.md §8).  One slab per GPU (real ranks) is the single-part case of §9e, where the
          // pipeline is measured to help at every size (20000x40000: 3.44 vs 3.75 ms per block).
          size_t free_b = 0, total_b = 0;
          CK(cudaMemGetInfo(&free_b, &total_b));
          mpipe = 2.2 * 8.0 * (double)v.rows * (double)v.ld * nslabs <= (double)free_b &&
                  (nslabs == 1 || 16.0 * (double)v.rows * (double)v.ld <= 2.5e9);
        }
      }
      // k_update_s: column chunks of cw doubles x row groups; all CTAs resident
      // (nc, cw, Gr) minimising the busiest CTA's share cw * ceil(rows / Gr) over the
      // occ * sms resident slots (pipelined: the SMs left over by the selection cluster),
      // chunks at least 3/4 of the consumer lanes wide (e.g. 37 chunks x 8 row groups =
      // 296 CTAs at 8000^2 instead of 32 x 9 = 288)
      const int cwmax = 2 * sx::kThreads;
      int occ = 1;
      pass_cfg = sx::pass_cfg_choice(overlap || mpipe, 16.0 * v.rows * v.ld);   // bytes read + written per pass
      CK(sx::update_s_occupancy(pass_cfg, look, &occ, sx::update_s_smem(pass_cfg, cwmax, v.rows, look)));
      if (occ < 1) return fail(SIMPLEX_E_CUDA, "rank-s pass kernel cannot be resident");
      const char* ps = sx::experiment_env("SIMPLEX_PASS_SMS");
      const long long slots = (long long)occ * (ps ? atoi(ps) : overlap ? sms - sl.look_grid
                                                                : mpipe ? sms - nslabs * sl.look_grid : sms);
      const long long nc0 = (v.ld + cwmax - 1) / cwmax;
      long long best = LLONG_MAX;
      for (long long nc = nc0; nc <= std::max(nc0, std::min(slots, 4 * nc0)); ++nc) {
        const long long cw = roundup((v.ld + nc - 1) / nc, 2);
        if (cw > cwmax || (cw < cwmax * 3 / 4 && nc > nc0)) continue;   // keep >= 3/4 of the lanes busy
        const long long gr = std::max(1LL, std::min<long long>(v.rows, slots / nc));
        const long long cost = cw * ((v.rows + gr - 1) / gr);
        if (cost < best) {
          best = cost;
          sl.nc = (int)nc;
          sl.cw = (int)cw;
          sl.Gr = (int)gr;
        }
      }
    }
    {
      // k_update (one pivot per pass; also the Phase I drive-out pivots): kUpdateCtasPerSm
      // CTAs per SM; thread t owns column pair t mod (ld/2)
      int occ = 1;
      CK(sx::update_occupancy(&occ));
      const long long tpr = v.ld / 2;                      // threads per row
      long long threads = (long long)std::min(occ, sx::kUpdateCtasPerSm) * sms * sx::kThreads;
      threads = std::max(threads, roundup(tpr, sx::kThreads));
      sl.q = (int)std::max(1LL, std::min<long long>(v.rows, threads / tpr));
      sl.upd_grid = (int)((sl.q * tpr + sx::kThreads - 1) / sx::kThreads);
    }

    RET(dalloc(&v.T, (size_t)v.rows * v.ld));
    RET(dalloc(&v.price, v.nslot));
    RET(dalloc(&v.col, v.rows + 2));
    RET(dalloc(&v.rownorm, v.ld));
    if (overlap || mpipe) RET(dalloc(&sl.T2, (size_t)v.rows * v.ld));
    RET(dalloc(&v.rcand, std::max(sl.sel_grid, sl.look_grid)));
    RET(dalloc(&v.basis, m));
    RET(dalloc(&v.art_of_row, m));
    RET(dalloc(&v.neg_rows, std::max<long long>(arts, 1)));
    RET(dalloc(&v.cvec, n));
    v.trace_cap = opt.record_trace ? cap : 0;
    RET(dalloc(&v.trace_k, std::max<long long>(v.trace_cap, 1)));
    RET(dalloc(&v.trace_r, std::max<long long>(v.trace_cap, 1)));
    RET(dalloc(&v.st, 1));
    CK(cudaMemsetAsync(v.st, 0, sizeof(sx::DevState), stream));   // xseq starts at 0 (never reset)
    if (look > 1) {
      RET(dalloc(&v.colS, (size_t)v.rows * sx::kColS));
      RET(dalloc(&v.prowS, (size_t)sx::kColS * v.ld));
      RET(dalloc(&v.colT, (size_t)v.rows * sx::kColS));
      RET(dalloc(&v.R0, v.ld));
      RET(dalloc(&v.RHS, v.rows));
      RET(dalloc(&v.pcand, sl.look_grid));
      if (nparts == 1 && !hybrid && !force_nccl) {
        // k_look2 when the own-bank chain operands fit in shared memory; the
        // experiment build can force k_lookahead (SIMPLEX_LOOK_V1=1)
        const char* e1 = sx::experiment_env("SIMPLEX_LOOK_V1");
        const long long hn = (e1 && e1[0] == '1') ? 0 : sx::look2_prepare(&v, sl.look_grid);
        if (hn > 0) RET(dalloc(&v.hand, (size_t)hn));
      }
      v.time_pass = time_pass() ? 1 : 0;
      if (sx::experiment_env("SIMPLEX_PROBE")) {          // experiment hook: selection phase stamps
        RET(dalloc(&v.probe, (size_t)sx::kProbeSlots * 16 * sx::kProbeEv));
        CK(cudaMemset(v.probe, 0, sizeof(unsigned long long) * sx::kProbeSlots * 16 * sx::kProbeEv));
      }
    }
  }
  if (hybrid) {
    RET(dalloc(&send, m + 3));
    RET(dalloc(&d_wcol, m + 1));
    CK(cudaHostAlloc(reinterpret_cast<void**>(&h_slot), sizeof(double) * (size_t)(m + 3), cudaHostAllocDefault));
    CK(cudaHostAlloc(reinterpret_cast<void**>(&h_wcol), sizeof(double) * (size_t)(m + 1), cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&ev_slot, cudaEventDisableTiming));
    wcol.resize((size_t)(m + 1));
  }
  RET(dalloc(&d_x, n));
  RET(dalloc(&d_y, m));
  RET(dalloc(&d_obj, 1));
  RET(dalloc(&d_b, m));
  RET(dalloc(&d_res, 4));
  if (small) RET(dalloc(&d_stage, (size_t)(m * n + m + n)));   // simplex_solve_lp's host-input staging
  CK(cudaHostAlloc(reinterpret_cast<void**>(&h_res), sizeof(double) * 4, cudaHostAllocDefault));
  RET(dalloc(&d_hash, 1));

  // ---- exchange buffers
  xstride = roundup(m + 3, 2);
  if (gathered()) {
    RET(dalloc(&recv, (size_t)(look > 1 ? 2 : 1) * nparts * xstride));   // look-ahead: two exchanges
    if (use_nccl() && !p2p) RET(dalloc(&send, xstride));
  }
  if (use_nccl()) {
    ncclUniqueId id;
    if (nranks > 1) {
      if (!opt.nccl_id) return fail(SIMPLEX_E_ARG, "nranks > 1 needs nccl_id");
      std::memcpy(&id, opt.nccl_id, sizeof(id));
    } else {
      NK(ncclGetUniqueId(&id));
    }
    NK(ncclCommInitRank(&comm, nranks, id, rank));
  }
  if (p2p) RET(setup_p2p());
  if (!p2p) mblock = mpipe = false;              // peers unreachable: NCCL per pivot
  if (mblock && nslabs > 1) {                     // selection streams (forked inside the graphs)
    xs.assign((size_t)nslabs, nullptr);
    ev_join.assign((size_t)nslabs, nullptr);
    for (int i = 0; i < nslabs; ++i) {
      CK(cudaStreamCreateWithFlags(&xs[(size_t)i], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ev_join[(size_t)i], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  }
  return SIMPLEX_OK;
}

// Peer-memory exchange of the multi-part look-ahead: every part's k_mlook stores
// its slot, as sequence-numbered LL words, straight into every rank's gather buffer.  Ranks map
// each other's gather buffer through CUDA IPC; the handles travel over NCCL once.  Falls back to
// the NCCL allgather (exchange = 0) when a peer is not reachable.
simplex_err simplex_s::setup_p2p() {
  const long long half = (long long)nparts * xstride;
  RET(dalloc(&xll, (size_t)(2 * 2 * half)));                            // 2 parities x 2 words per value
  CK(cudaMemsetAsync(xll, 0, sizeof(unsigned long long) * 2 * 2 * half, stream));   // sequence 0: never written
  std::vector<unsigned long long*> px((size_t)nranks, xll);
  if (nranks > 1) {
    int ok = 1;
    std::vector<int> devs((size_t)nranks, -1);
    {
      int* d_dev = nullptr;
      RET(dalloc(&d_dev, (size_t)nranks));
      CK(cudaMemcpyAsync(d_dev + rank, &device, sizeof(int), cudaMemcpyHostToDevice, stream));
      NK(ncclAllGather(d_dev + rank, d_dev, 1, ncclInt32, comm, stream));
      CK(cudaMemcpyAsync(devs.data(), d_dev, sizeof(int) * nranks, cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
    }
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) continue;
      int can = 0;
      if (devs[r] == device || cudaDeviceCanAccessPeer(&can, device, devs[r]) != cudaSuccess) can = 0;
      ok &= can;
    }
    cudaGetLastError();
    // every rank must take the same decision
    {
      int* d_ok = nullptr;
      RET(dalloc(&d_ok, 1));
      CK(cudaMemcpyAsync(d_ok, &ok, sizeof(int), cudaMemcpyHostToDevice, stream));
      NK(ncclAllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, comm, stream));
      CK(cudaMemcpyAsync(&ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
    }
    if (!ok) {
      if (opt.exchange >= 2) return fail(SIMPLEX_E_CUDA, "exchange = 2/3 (peer memory) but a peer GPU is not reachable");
      p2p = false;
      RET(dalloc(&send, xstride));                        // NCCL allgather path
      return SIMPLEX_OK;
    }
    cudaIpcMemHandle_t hx;
    CK(cudaIpcGetMemHandle(&hx, xll));
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    unsigned char* d_h = nullptr;
    RET(dalloc(&d_h, hb * nranks));
    std::vector<unsigned char> hh(hb * nranks);
    std::memcpy(hh.data() + hb * rank, &hx, sizeof(hx));
    CK(cudaMemcpyAsync(d_h + hb * rank, hh.data() + hb * rank, hb, cudaMemcpyHostToDevice, stream));
    NK(ncclAllGather(d_h + hb * rank, d_h, hb, ncclUint8, comm, stream));
    CK(cudaMemcpyAsync(hh.data(), d_h, hb * nranks, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    int opened = 1;                                  // every rank must agree that every mapping worked
    for (int r = 0; r < nranks && opened; ++r) {
      if (r == rank) continue;
      cudaIpcMemHandle_t a;
      std::memcpy(&a, hh.data() + hb * r, sizeof(a));
      void* pa = nullptr;
      if (cudaIpcOpenMemHandle(&pa, a, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        opened = 0;
        break;
      }
      ipc_open.push_back(pa);
      px[(size_t)r] = static_cast<unsigned long long*>(pa);
    }
    {
      int* d_op = reinterpret_cast<int*>(d_h);
      CK(cudaMemcpyAsync(d_op, &opened, sizeof(int), cudaMemcpyHostToDevice, stream));
      NK(ncclAllReduce(d_op, d_op, 1, ncclInt32, ncclMin, comm, stream));
      CK(cudaMemcpyAsync(&opened, d_op, sizeof(int), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
    }
    if (!opened) {                                   // a CUDA-IPC mapping failed somewhere: NCCL instead
      for (void* pa : ipc_open) cudaIpcCloseMemHandle(pa);
      ipc_open.clear();
      if (opt.exchange >= 2) return fail(SIMPLEX_E_CUDA, "exchange = 2/3 (peer memory) but a CUDA-IPC mapping failed");
      p2p = false;
      RET(dalloc(&send, xstride));
      return SIMPLEX_OK;
    }
    // no rank may store into a peer before that peer's buffer is zeroed: the memset above is
    // ordered before this allreduce on every rank
    NK(ncclAllReduce(reinterpret_cast<int*>(d_h), reinterpret_cast<int*>(d_h), 1, ncclInt32, ncclMax, comm, stream));
    CK(cudaStreamSynchronize(stream));
  }
  xpeers.assign((size_t)nslabs, sx::XPeers{});
  for (int sidx = 0; sidx < nslabs; ++sidx) {
    sx::XPeers& xp = xpeers[(size_t)sidx];
    xp.n = nranks;
    xp.part = rank * nslabs + sidx;
    xp.half = half;
    for (int r = 0; r < nranks; ++r) xp.x[r] = px[(size_t)r];
    xp.mine = xll;
    xp.timeout_ns = 1000000ull * (unsigned long long)(opt.exchange_timeout_ms > 0 ? opt.exchange_timeout_ms : 30000);
  }
  return SIMPLEX_OK;
}

simplex_err simplex_s::load(const double* A, const double* b, const double* c, bool first) {
  if (!A || !b || !c) return fail(SIMPLEX_E_ARG, "NULL input pointer");
  RET(enter());
  // the row map of b's signs (Phase I): scanned on the host at create and on a reset of a Phase I
  // handle; a handle without artificials keeps its all-slack map and k_build flags any b_i < 0
  // (kErrNegRhs) — a reset then costs one host synchronisation
  std::vector<int> art_of_row, neg;
  const bool remap = first || arts > 0;
  if (remap) {
    RET(scan_b(b, &art_of_row, &neg));
    if ((long long)neg.size() != arts)
      return fail(SIMPLEX_E_ARG, "reset: the number of negative b entries differs from create's");
    art_rows = neg;
  }
  CK(cudaMemcpyAsync(d_b, b, sizeof(double) * m, cudaMemcpyDefault, stream));
  for (auto& sl : slabs) {
    sx::SlabView& v = sl.v;
    if (remap) CK(cudaMemcpyAsync(v.art_of_row, art_of_row.data(), sizeof(int) * m, cudaMemcpyHostToDevice, stream));
    if (remap && arts > 0) CK(cudaMemcpyAsync(v.neg_rows, neg.data(), sizeof(int) * arts, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(v.cvec, c, sizeof(double) * n, cudaMemcpyDefault, stream));
    const long long ns = std::max<long long>(0, std::min<long long>(v.c0 + v.w, n) - v.c0);  // structural cols
    if (ns > 0) {
      // A's slab columns straight into rows 1..m (pitched copy), c's into row 0
      CK(cudaMemcpy2DAsync(v.T + v.ld, sizeof(double) * v.ld, A + v.c0, sizeof(double) * n,
                           sizeof(double) * ns, m, cudaMemcpyDefault, stream));
      CK(cudaMemcpyAsync(v.T, c + v.c0, sizeof(double) * ns, cudaMemcpyDefault, stream));
    }
    CK(sx::launch_init_state(v, n, cap, stream));
    CK(sx::launch_build(v, d_b, n, stream, sms));
    if (arts > 0) CK(sx::launch_phase1_row0(v, stream));     // Phase I objective (reading p2)
    CK(sx::launch_price0(v, opt.tol_opt, stream));
  }
  kernel_launches += (3 + (arts > 0 ? 1 : 0)) * nslabs;
  if (hybrid) RET(load_lane(A, b, c));
  // validation result: every slab's error bits, one synchronisation (which also keeps the host
  // vectors above alive until their copies have run)
  for (int s = 0; s < nslabs; ++s)
    CK(cudaMemcpyAsync(&h_err[s], &slabs[s].v.st->err, sizeof(unsigned int), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  unsigned int err = 0;
  for (int s = 0; s < nslabs; ++s) err |= h_err[s];
  if (use_nccl()) {
    // every rank must agree on the verdict (each checked only its own columns)
    unsigned int* d_err = reinterpret_cast<unsigned int*>(d_hash);
    CK(cudaMemcpyAsync(d_err, &err, sizeof(err), cudaMemcpyHostToDevice, stream));
    NK(ncclAllReduce(d_err, d_err, 1, ncclUint32, ncclMax, comm, stream));
    CK(cudaMemcpyAsync(&h_state[2].err, d_err, sizeof(err), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    err = h_state[2].err;
  }
  status = SIMPLEX_RUNNING;
  slot_ready = false;
  phase = arts > 0 ? 1 : 2;
  drive_pending = false;
  drive_done = 0;
  drive_rows.clear();
  it = 0;
  if (err & sx::kErrNonFinite) return fail(SIMPLEX_E_NONFINITE, "A, b or c contains NaN or Inf");
  if (err & sx::kErrNegRhs)
    return fail(SIMPLEX_E_ARG, "reset: the number of negative b entries differs from create's");
  return SIMPLEX_OK;
}

simplex_err simplex_s::enqueue_pivot(int slot, int t) {
  if (look > 1 && gathered()) {
    // multi-part rank-s block: k_mlook for the block start and for every pivot on every part,
    // each followed by the exchange of the parts' candidate columns (exchange e in buffer e&1),
    // then the pass on every part's slab
    if (mpipe) {
      // multi-part pipeline (the §9e scheme on P parts): block t's starting tableau is in buffer
      // t&1 of every slab and its pivots in bank t&1; select block t+1 (chaining block t first)
      // on the selection streams WHILE block t's slab passes (buffer t&1 -> the other) run here
      // One stream, programmatic dependent launch (as in §9e): the first part's selection is a
      // normal launch (everything before it has finished), the other parts' selections and then
      // the slab passes are launched behind it without waiting, so every selection cluster is
      // placed before the passes fill the remaining SMs.  The pass times itself on the device
      // (time_kernels) because event nodes would serialize it after the selections.
      const int q = t & 1;
      for (int sidx = 0; sidx < nslabs; ++sidx) {
        const Slab& sl = slabs[sidx];
        CK(sx::launch_mblock(sl.v, q ? sl.T2 : sl.v.T, nparts, xstride, look, q ^ 1, q, opt.tol_opt, opt.tol_piv,
                             sl.look_grid, xpeers[(size_t)sidx], stream, sidx > 0));
      }
      for (auto& sl : slabs) {
        double* buf[2] = {sl.v.T, sl.T2};
        CK(sx::launch_update_s(pass_cfg, sl.v, look, buf[q], buf[q ^ 1], q, sl.nc, sl.Gr, sl.cw, stream, true));
      }
      return SIMPLEX_OK;
    }
    if (mblock) {
      // the block's selection: one k_mblock per part (virtual slabs concurrently), then the passes
      RET(mselect(0, 0, -1, true));
      if (opt.time_kernels) CK(cudaEventRecordWithFlags(tev[slot][2 * t], stream, cudaEventRecordExternal));
      for (auto& sl : slabs)
        CK(sx::launch_update_s(pass_cfg, sl.v, look, sl.v.T, sl.v.T, 0, sl.nc, sl.Gr, sl.cw, stream, false));
      if (opt.time_kernels) CK(cudaEventRecordWithFlags(tev[slot][2 * t + 1], stream, cudaEventRecordExternal));
      return SIMPLEX_OK;
    }
    double* X[2] = {recv, recv + (long long)nparts * xstride};
    static const sx::XPeers no_peers{};
    for (int u = -1; u < look; ++u) {
      for (int sidx = 0; sidx < nslabs; ++sidx) {
        const Slab& sl = slabs[sidx];
        double* xout = p2p ? nullptr : use_nccl() ? send : X[(u + 1) & 1] + (long long)sidx * xstride;
        CK(sx::launch_mlook(sl.v, u >= 0 ? X[u & 1] : nullptr, xout, nparts, xstride, u, look, opt.tol_opt,
                            opt.tol_piv, sl.look_grid, p2p ? xpeers[(size_t)sidx] : no_peers, stream));
      }
      if (!p2p && use_nccl() && u + 1 < look)
        NK(ncclAllGather(send, X[(u + 1) & 1], (size_t)xstride, ncclFloat64, comm, stream));
    }
    if (opt.time_kernels) CK(cudaEventRecordWithFlags(tev[slot][2 * t], stream, cudaEventRecordExternal));
    for (auto& sl : slabs)
      CK(sx::launch_update_s(pass_cfg, sl.v, look, sl.v.T, sl.v.T, 0, sl.nc, sl.Gr, sl.cw, stream, false));
    if (opt.time_kernels) CK(cudaEventRecordWithFlags(tev[slot][2 * t + 1], stream, cudaEventRecordExternal));
    return SIMPLEX_OK;
  }
  if (look > sx::kMaxLook) {
    // pair schedule: bank 0 selected from the tableau, bank 1 from the same tableau chaining
    // bank 0 first (the pipeline's mode of k_lookahead), then one pass of up to 32 chains
    const Slab& sl = slabs[0];
    CK(sx::launch_lookahead(sl.v, sl.v.T, sx::kMaxLook, 0, -1, opt.tol_opt, opt.tol_piv, sl.look_grid, false, stream));
    CK(sx::launch_lookahead(sl.v, sl.v.T, look - sx::kMaxLook, 1, 0, opt.tol_opt, opt.tol_piv, sl.look_grid,
                            look_cache, stream));
    if (opt.time_kernels) CK(cudaEventRecordWithFlags(tev[slot][2 * t], stream, cudaEventRecordExternal));
    CK(sx::launch_update_s(pass_cfg, sl.v, look, sl.v.T, sl.v.T, 0, sl.nc, sl.Gr, sl.cw, stream, pdl && !opt.time_kernels));
    if (opt.time_kernels) CK(cudaEventRecordWithFlags(tev[slot][2 * t + 1], stream, cudaEventRecordExternal));
    return SIMPLEX_OK;
  }
  if (look > 1) {
    const Slab& sl = slabs[0];
    if (overlap) {
      // software pipeline: block t's starting tableau is in buffer t&1 and its
      // pivots in chain bank t&1.  Select block t+1 (chaining block t first) into the other
      // bank on the cluster, and let block t's pass (buffer t&1 -> the other) start on the
      // remaining SMs as soon as the cluster is resident (PDL; it does not wait for it).
      const int q = t & 1;
      double* buf[2] = {sl.v.T, sl.T2};
      static const bool time_sel = sx::experiment_env("SIMPLEX_TIME_SELECT") != nullptr;   // experiment hook
      if (opt.time_kernels && !time_sel) {
        // the pass times itself on the device (SlabView::time_pass) so that it still runs
        // concurrently with the selection: the production launch sequence, no event nodes
        CK(sx::launch_lookahead(sl.v, buf[q], look, q ^ 1, q, opt.tol_opt, opt.tol_piv, sl.look_grid, look_cache,
                                stream));
        CK(sx::launch_update_s(pass_cfg, sl.v, look, buf[q], buf[q ^ 1], q, sl.nc, sl.Gr, sl.cw, stream, pdl));
        return SIMPLEX_OK;
      }
      if (opt.time_kernels && time_sel) CK(cudaEventRecordWithFlags(tev[slot][2 * t], stream, cudaEventRecordExternal));
      CK(sx::launch_lookahead(sl.v, buf[q], look, q ^ 1, q, opt.tol_opt, opt.tol_piv, sl.look_grid, look_cache, stream));
      if (opt.time_kernels)
        CK(cudaEventRecordWithFlags(tev[slot][2 * t + (time_sel ? 1 : 0)], stream, cudaEventRecordExternal));
      if (opt.time_kernels && time_sel) {
        CK(sx::launch_update_s(pass_cfg, sl.v, look, buf[q], buf[q ^ 1], q, sl.nc, sl.Gr, sl.cw, stream, false));
        return SIMPLEX_OK;
      }
      CK(sx::launch_update_s(pass_cfg, sl.v, look, buf[q], buf[q ^ 1], q, sl.nc, sl.Gr, sl.cw, stream,
                             pdl && !opt.time_kernels));
      if (opt.time_kernels) CK(cudaEventRecordWithFlags(tev[slot][2 * t + 1], stream, cudaEventRecordExternal));
      return SIMPLEX_OK;
    }
    // rank-s block: select up to `look` pivots ahead, then one pass applies them all in place
    CK(sx::launch_lookahead(sl.v, sl.v.T, look, 0, -1, opt.tol_opt, opt.tol_piv, sl.look_grid, false, stream));
    if (opt.time_kernels) CK(cudaEventRecordWithFlags(tev[slot][2 * t], stream, cudaEventRecordExternal));
    CK(sx::launch_update_s(pass_cfg, sl.v, look, sl.v.T, sl.v.T, 0, sl.nc, sl.Gr, sl.cw, stream, pdl && !opt.time_kernels));
    if (opt.time_kernels) CK(cudaEventRecordWithFlags(tev[slot][2 * t + 1], stream, cudaEventRecordExternal));
    return SIMPLEX_OK;
  }
  // PDL (programmatic dependent launch) only between two of our kernels: not after an
  // NCCL collective or an event-record node.
  bool prev_is_ours = t > 0;   // previous node in the segment: k_update of the last pivot
  if (gathered()) {
    if (use_nccl()) {
      CK(sx::launch_pack(slabs[0].v, send, slabs[0].sel_grid, stream, pdl && prev_is_ours && !opt.time_kernels));
      NK(ncclAllGather(send, recv, (size_t)xstride, ncclFloat64, comm, stream));
      prev_is_ours = false;
    } else {
      for (int s = 0; s < nslabs; ++s) {
        CK(sx::launch_pack(slabs[s].v, recv + (long long)s * xstride, slabs[s].sel_grid, stream,
                           pdl && prev_is_ours && !opt.time_kernels));
        prev_is_ours = true;
      }
    }
  }
  const sx::XView x = xview();
  for (auto& sl : slabs) {
    CK(sx::launch_select(sl.v, x, opt.tol_piv, sl.sel_grid, stream, pdl && prev_is_ours && !opt.time_kernels));
    prev_is_ours = true;
  }
  if (opt.time_kernels) CK(cudaEventRecordWithFlags(tev[slot][2 * t], stream, cudaEventRecordExternal));
  for (auto& sl : slabs) {
    CK(sx::launch_update(sl.v, sl.q, opt.tol_opt, sl.upd_grid, stream, pdl && !opt.time_kernels));
  }
  if (opt.time_kernels) CK(cudaEventRecordWithFlags(tev[slot][2 * t + 1], stream, cudaEventRecordExternal));
  return SIMPLEX_OK;
}

simplex_err simplex_s::build_graphs() {
  if (graphs_ready) return SIMPLEX_OK;
  for (int slot = 0; slot < 2; ++slot) {
    if (opt.time_kernels) {
      tev[slot].resize(2 * steps_per_segment());
      for (auto& e : tev[slot]) CK(cudaEventCreate(&e));
    }
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    simplex_err e = SIMPLEX_OK;
    for (int t = 0; t < steps_per_segment() && e == SIMPLEX_OK; ++t) e = enqueue_pivot(slot, t);
    if (e == SIMPLEX_OK) {
      cudaError_t ce = cudaMemcpyAsync(&h_state[slot], slabs[0].v.st, sizeof(sx::DevState),
                                       cudaMemcpyDeviceToHost, stream);
      if (ce != cudaSuccess) e = fail(SIMPLEX_E_CUDA, std::string("capture memcpy: ") + cudaGetErrorString(ce));
    }
    cudaError_t ce = cudaStreamEndCapture(stream, &g);
    if (e != SIMPLEX_OK) {
      if (g) cudaGraphDestroy(g);
      return e;
    }
    if (ce != cudaSuccess) return fail(SIMPLEX_E_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(ce));
    ce = cudaGraphInstantiate(&seg[slot], g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return fail(SIMPLEX_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ce));
  }
  graphs_ready = true;
  return SIMPLEX_OK;
}

simplex_err simplex_s::run(long long max_pivots, long long* done) {
  const long long it0 = it;
  if (done) *done = 0;
  if (status != SIMPLEX_RUNNING) return SIMPLEX_OK;
  if (small) return run_small(max_pivots, done);
  if (hybrid) return run_hybrid(max_pivots, done);
  RET(build_graphs());
  RET(enter());
  const long long stop_at = max_pivots > 0 ? it + max_pivots : LLONG_MAX;
  for (auto& sl : slabs) CK(sx::launch_set_stop(sl.v.st, stop_at, stream));
  kernel_launches += nslabs;
  CK(cudaEventRecord(ev_loop0, stream));
  bool skip_loop = false;
  if (drive_pending) {                            // a Phase I drive-out stopped by the last call
    RET(phase_transition());
    skip_loop = status != SIMPLEX_RUNNING || it >= stop_at || drive_pending;
  }
  for (; !skip_loop;) {
    if (overlap) {
      // pipeline prologue: the first block is selected from the current tableau into bank 0
      const Slab& sl = slabs[0];
      CK(sx::launch_lookahead(sl.v, sl.v.T, look, 0, -1, opt.tol_opt, opt.tol_piv, sl.look_grid, false, stream));
      ++kernel_launches;
    }
    if (mpipe) {                                  // multi-part pipeline prologue (bank 0, buffer 0)
      RET(mselect(0, 0, -1, true));
      kernel_launches += nslabs;
    }
    long long launched = 0, completed = 0, seen = it;
    bool stop = false;
    for (;;) {
      while (!stop && launched - completed < 2) {
        const int slot = (int)(launched & 1);
        CK(cudaGraphLaunch(seg[slot], stream));
        CK(cudaEventRecord(ev_done[slot], stream));
        ++launched;
        ++graph_launches;
        kernel_launches += kernels_per_segment();
      }
      const int slot = (int)(completed & 1);
      CK(cudaEventSynchronize(ev_done[slot]));
      const sx::DevState hs = h_state[slot];
      ++completed;
      const long long piv = hs.it - seen;
      if (opt.time_kernels && time_pass()) {            // device-side pass timer (cumulative)
        upd_ms = hs.pass_ns / 1e6;
        upd_launches = hs.pass_n;
      } else if (opt.time_kernels) {
        const long long passes = look > 1 ? (piv + look - 1) / look : piv;   // k_update launches that did work
        for (long long q = 0; q < passes && q < steps_per_segment(); ++q) {
          float ms = 0.f;
          CK(cudaEventElapsedTime(&ms, tev[slot][2 * q], tev[slot][2 * q + 1]));
          upd_ms += ms;
          ++upd_launches;
        }
      }
      if (hs.err & sx::kErrExchange) {
        cudaStreamSynchronize(stream);
        faulted = true;
        return fail(SIMPLEX_E_NCCL, "peer-memory exchange timed out: a peer did not publish its candidate "
                                    "column within exchange_timeout_ms (the handle must be destroyed)");
      }
      seen = hs.it;
      status = hs.status;
      it = hs.it;
      if (hs.status != SIMPLEX_RUNNING || hs.it >= stop_at) stop = true;
      if (stop && completed == launched) break;
    }
    if (overlap) {
      // pipeline drain: the last selected block (bank 0) is applied in place to buffer 0
      const Slab& sl = slabs[0];
      CK(sx::launch_update_s(pass_cfg, sl.v, look, sl.v.T, sl.v.T, 0, sl.nc, sl.Gr, sl.cw, stream, false));
      ++kernel_launches;
    }
    if (mpipe) {                                  // multi-part pipeline drain
      for (auto& sl : slabs)
        CK(sx::launch_update_s(pass_cfg, sl.v, look, sl.v.T, sl.v.T, 0, sl.nc, sl.Gr, sl.cw, stream, false));
      kernel_launches += nslabs;
    }
    // Phase I optimal: decide feasibility, drive artificials out, install the objective
    if (status == SIMPLEX_OPTIMAL && phase == 1) {
      RET(phase_transition());
      if (status == SIMPLEX_RUNNING && it < stop_at) continue;
    }
    break;
  }
  CK(cudaEventRecord(ev_loop1, stream));
  CK(cudaEventSynchronize(ev_loop1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ev_loop0, ev_loop1));
  loop_ms += ms;
  if (done) *done = it - it0;
  return SIMPLEX_OK;
}

// The latency path: one k_solve_small launch runs pivots until a terminal status or stop_at.
simplex_err simplex_s::run_small(long long max_pivots, long long* done) {
  const long long it0 = it;
  RET(enter());
  const long long stop_at = max_pivots > 0 ? it + max_pivots : LLONG_MAX;
  const sx::SlabView& v = slabs[0].v;
  CK(cudaEventRecord(ev_loop0, stream));
  CK(sx::launch_solve_small(v, stop_at, opt.tol_opt, opt.tol_piv, stream));
  CK(cudaEventRecord(ev_loop1, stream));
  CK(cudaMemcpyAsync(&h_state[2], v.st, sizeof(sx::DevState), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  ++kernel_launches;
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ev_loop0, ev_loop1));
  loop_ms += ms;
  if (opt.time_kernels) {
    upd_ms += ms;
    ++upd_launches;
  }
  status = h_state[2].status;
  it = h_state[2].it;
  if (done) *done = it - it0;
  return SIMPLEX_OK;
}

// simplex_solve_lp on the latency path: ONE launch builds Table I from A, b, c, solves and extracts
// (k_solve_small's LP mode), ONE host synchronisation — reset + solve + get_solution of a small LP
// without the three calls' separate round trips (small LPs are overhead-bound).
static bool on_device(const void* p, int dev) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) && a.device == dev;
}

simplex_err simplex_s::solve_lp_small(const double* A, const double* b, const double* c, double* x, double* y,
                                      double* objective, long long* pivots) {
  RET(enter());
  const double* dA = A;
  const double* db = b;
  const double* dc = c;
  const bool ha = !on_device(A, device), hb = !on_device(b, device), hc = !on_device(c, device);
  if (ha || hb || hc) {
    if (!d_stage) RET(dalloc(&d_stage, (size_t)(m * n + m + n)));
    if (ha) CK(cudaMemcpyAsync(d_stage, A, sizeof(double) * m * n, cudaMemcpyDefault, stream));
    if (hb) CK(cudaMemcpyAsync(d_stage + m * n, b, sizeof(double) * m, cudaMemcpyDefault, stream));
    if (hc) CK(cudaMemcpyAsync(d_stage + m * n + m, c, sizeof(double) * n, cudaMemcpyDefault, stream));
    if (ha) dA = d_stage;
    if (hb) db = d_stage + m * n;
    if (hc) dc = d_stage + m * n + m;
  }
  // outputs on this device are written by the kernel itself (no copies)
  const bool dx = x && on_device(x, device), dy = y && on_device(y, device);
  const sx::SmallLP io{dA, db, dc, n, dx ? x : d_x, dy ? y : d_y, d_res};
  CK(sx::launch_solve_small(slabs[0].v, LLONG_MAX, opt.tol_opt, opt.tol_piv, stream, io));
  ++kernel_launches;
  if (x && !dx) CK(cudaMemcpyAsync(x, d_x, sizeof(double) * n, cudaMemcpyDefault, stream));
  if (y && !dy) CK(cudaMemcpyAsync(y, d_y, sizeof(double) * m, cudaMemcpyDefault, stream));
  CK(cudaMemcpyAsync(h_res, d_res, sizeof(double) * 4, cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  slot_ready = false;
  phase = 2;
  drive_pending = false;
  drive_done = 0;
  drive_rows.clear();
  const unsigned int err = (unsigned int)h_res[3];
  status = SIMPLEX_RUNNING;
  it = 0;
  if (err & sx::kErrNonFinite) return fail(SIMPLEX_E_NONFINITE, "A, b or c contains NaN or Inf");
  if (err & sx::kErrNegRhs) return fail(SIMPLEX_E_ARG, "reset: the number of negative b entries differs from create's");
  status = (int)h_res[1];
  it = (long long)h_res[2];
  if (objective) *objective = h_res[0];
  if (pivots) *pivots = it;
  return SIMPLEX_OK;
}

// ---- hybrid CPU lane (options.host_share, §IV)
// The host lane's columns (host memory) from the caller's A / b / c (host or device pointers).
simplex_err simplex_s::load_lane(const double* A, const double* b, const double* c) {
  const long long ncols_a = std::max(0LL, std::min(n, lane.c0 + lane.hw) - lane.c0);
  std::vector<double> Acols((size_t)(m * std::max(ncols_a, 1LL))), hb((size_t)m), hc((size_t)n);
  if (ncols_a > 0)
    CK(cudaMemcpy2DAsync(Acols.data(), sizeof(double) * ncols_a, A + lane.c0, sizeof(double) * n,
                         sizeof(double) * ncols_a, m, cudaMemcpyDefault, stream));
  CK(cudaMemcpyAsync(hb.data(), b, sizeof(double) * m, cudaMemcpyDefault, stream));
  CK(cudaMemcpyAsync(hc.data(), c, sizeof(double) * n, cudaMemcpyDefault, stream));
  CK(cudaStreamSynchronize(stream));
  if (!lane.build(Acols.data(), ncols_a, hc.data(), hb.data()))
    return fail(SIMPLEX_E_NONFINITE, "A, b or c contains NaN or Inf");
  host_ms = host_wait_ms = 0.0;
  return SIMPLEX_OK;
}

// The GPU part's Step-1 candidate and its column: write back any deferred pivot row, fold the
// per-warp candidates (k_pack: [v, k, col[0..m]]), copy the slot to pinned host memory.
simplex_err simplex_s::enqueue_gpu_candidate() {
  const Slab& sl = slabs[0];
  CK(sx::launch_pack(sl.v, send, 1, stream, false));
  CK(cudaMemcpyAsync(h_slot, send, sizeof(double) * (size_t)(m + 3), cudaMemcpyDeviceToHost, stream));
  CK(cudaEventRecord(ev_slot, stream));
  ++kernel_launches;
  slot_ready = true;
  return SIMPLEX_OK;
}

// One pivot per iteration, the paper's per-iteration schedule: both lanes'
// Step-1 candidates are folded on the host (the paper's "compared ... global maximum index"),
// the ratio test runs on the host against the replicated rhs, and then the GPU applies the pivot
// to its columns (k_flush, k_force with the winning column, k_update, and already the next
// candidate: k_pack + D2H) WHILE the host cores apply it to theirs.  One host wait per pivot.
simplex_err simplex_s::run_hybrid(long long max_pivots, long long* done) {
  const long long it0 = it;
  RET(enter());
  const long long stop_at = max_pivots > 0 ? it + max_pivots : LLONG_MAX;
  const Slab& sl = slabs[0];
  CK(cudaEventRecord(ev_loop0, stream));
  if (!slot_ready) RET(enqueue_gpu_candidate());
  sx::HostCand hc = lane.candidate(opt.tol_opt);
  auto now_ms = []() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  while (status == SIMPLEX_RUNNING && it < stop_at) {
    const double t0 = now_ms();
    CK(cudaEventSynchronize(ev_slot));
    host_wait_ms += now_ms() - t0;
    sx::HostCand g{h_slot[0], 0};
    std::memcpy(&g.idx, &h_slot[1], sizeof(g.idx));
    const bool gpu_wins = g.v < hc.v || (g.v == hc.v && g.idx < hc.idx);
    const sx::HostCand win = gpu_wins ? g : hc;
    if (win.idx == LLONG_MAX) {                                            // Step 1: optimal
      status = SIMPLEX_OPTIMAL;
      break;
    }
    const long long k = win.idx;
    if (gpu_wins) std::memcpy(wcol.data(), h_slot + 2, sizeof(double) * (size_t)(m + 1));
    else lane.column(k, wcol.data());
    const sx::HostCand rb = lane.ratio(wcol.data(), opt.tol_piv);          // Step 2
    if (rb.idx == LLONG_MAX) {
      status = SIMPLEX_UNBOUNDED;
      break;
    }
    if (it >= cap) {                                                       // reading c12
      status = SIMPLEX_ITERATION_LIMIT;
      break;
    }
    const long long r = rb.idx & 0xffffffffLL;
    // Step 3 on the GPU's columns (asynchronous), then on the host lane's
    const double* dcol = send + 2;
    if (!gpu_wins) {
      std::memcpy(h_wcol, wcol.data(), sizeof(double) * (size_t)(m + 1));
      CK(cudaMemcpyAsync(d_wcol, h_wcol, sizeof(double) * (size_t)(m + 1), cudaMemcpyHostToDevice, stream));
      dcol = d_wcol;
    }
    CK(sx::launch_flush(sl.v, stream));
    CK(sx::launch_force(sl.v, (int)r, (int)k, dcol, stream));
    CK(sx::launch_update(sl.v, sl.q, opt.tol_opt, sl.upd_grid, stream, false));
    kernel_launches += 3;
    RET(enqueue_gpu_candidate());
    const double t1 = now_ms();
    lane.pivot(r, k, wcol.data());
    hc = lane.candidate(opt.tol_opt);
    host_ms += now_ms() - t1;
    ++it;
  }
  if (status != SIMPLEX_RUNNING) {
    CK(sx::launch_set_status(sl.v.st, status, stream));
    ++kernel_launches;
  }
  CK(cudaEventRecord(ev_loop1, stream));
  CK(cudaEventSynchronize(ev_loop1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ev_loop0, ev_loop1));
  loop_ms += ms;
  if (done) *done = it - it0;
  return SIMPLEX_OK;
}

// Phase I -> Phase II (readings p3-p5 of DESIGN.md), between device loops, on every column part:
// infeasible iff the Phase I optimum < -1e-7; each artificial still basic (rows ascending) is
// pivoted out on its first column j < n+m with |T[i][j]| > tol_piv over ALL parts (reading p4) —
// chosen, staged and applied on the device (kernels.cu k_drive_*, then the update kernel), with
// no host round trip per drive-out pivot; then the Phase II objective row is priced out on the
// device.  The only synchronisations: one to read the verdict and the basis when Phase I ends,
// one after the whole drive-out.  A drive-out that reaches stop_at (simplex_iterate) stays
// pending (DevState.drive_next) and resumes at the next call.
simplex_err simplex_s::phase_transition() {
  if (!drive_pending) {
    RET(flush_all());
    sx::SlabView& v0 = slabs[0].v;
    std::vector<int> basis((size_t)m);
    CK(cudaMemcpyAsync(&h_state[2].p, v0.T + v0.w, sizeof(double), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(basis.data(), v0.basis, sizeof(int) * m, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (h_state[2].p < -1e-7) {
      phase = 2;
      status = SIMPLEX_INFEASIBLE;
      for (auto& sl : slabs) CK(sx::launch_set_status(sl.v.st, SIMPLEX_INFEASIBLE, stream));
      CK(cudaStreamSynchronize(stream));
      return SIMPLEX_OK;
    }
    drive_rows.clear();
    for (long long i = 1; i <= m; ++i)
      if (basis[(size_t)(i - 1)] >= n + m) drive_rows.push_back((int)i);
    drive_pending = true;
    drive_done = 0;
    if (!d_fj) {
      RET(dalloc(&d_fj, (size_t)nslabs + 1));                     // per part + the minimum
      RET(dalloc(&d_fcol, (size_t)nranks * xcol_stride()));     // staged [flag, column] per rank
    }
    for (auto& sl : slabs) CK(sx::launch_set_status(sl.v.st, SIMPLEX_RUNNING, stream));
  }
  const bool multi = nparts > 1;
  const long long xs = xcol_stride();
  long long* fjmin = d_fj + nslabs;
  double* xmine = d_fcol + (long long)rank * xs;
  for (size_t q = (size_t)drive_done; q < drive_rows.size(); ++q) {
    const int i = drive_rows[q];
    for (int p = 0; p < nslabs; ++p)
      CK(sx::launch_drive_find(slabs[(size_t)p].v, i, n + m, opt.tol_piv, d_fj + p, stream));
    CK(sx::launch_drive_pick(d_fj, nslabs, fjmin, stream));
    if (nranks > 1) NK(ncclAllReduce(fjmin, fjmin, 1, ncclInt64, ncclMin, comm, stream));
    if (multi) {
      CK(cudaMemsetAsync(xmine, 0, sizeof(double), stream));
      for (auto& sl : slabs) CK(sx::launch_drive_col(sl.v, fjmin, xmine, stream));
      if (nranks > 1) NK(ncclAllGather(xmine, d_fcol, (size_t)xs, ncclFloat64, comm, stream));
    }
    for (auto& sl : slabs) {
      CK(sx::launch_drive_force(sl.v, i, (int)q, fjmin, multi ? (nranks > 1 ? d_fcol : xmine) : nullptr,
                                multi ? (nranks > 1 ? nranks : 1) : 0, xs, stream));
      CK(sx::launch_update(sl.v, sl.q, opt.tol_opt, sl.upd_grid, stream, false));
      CK(sx::launch_flush(sl.v, stream));
    }
    kernel_launches += 2 + 3 * nslabs + (multi ? nslabs : 0);
  }
  CK(cudaMemcpyAsync(&h_state[2], slabs[0].v.st, sizeof(sx::DevState), cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
  it = h_state[2].it;
  drive_done = h_state[2].drive_next;
  if (h_state[2].status == SIMPLEX_ITERATION_LIMIT) {
    status = SIMPLEX_ITERATION_LIMIT;
    drive_pending = false;
    phase = 2;
    return SIMPLEX_OK;
  }
  if (drive_done < (long long)drive_rows.size()) {     // stopped at stop_at: resume next call
    status = SIMPLEX_RUNNING;
    return SIMPLEX_OK;
  }
  drive_pending = false;
  phase = 2;
  for (auto& sl : slabs) {
    CK(sx::launch_phase2_row0(sl.v, n, stream));
    CK(sx::launch_price0(sl.v, opt.tol_opt, stream));
    CK(sx::launch_set_status(sl.v.st, SIMPLEX_RUNNING, stream));
  }
  kernel_launches += 3 * nslabs;
  CK(cudaStreamSynchronize(stream));
  status = SIMPLEX_RUNNING;
  return SIMPLEX_OK;
}

simplex_err simplex_s::flush_all() {
  for (auto& sl : slabs) CK(sx::launch_flush(sl.v, stream));
  kernel_launches += nslabs;
  return SIMPLEX_OK;
}

void simplex_s::release() {
  if (device >= 0) cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  if (const char* path = sx::experiment_env("SIMPLEX_PROBE"))   // experiment hook: dump the stamps
    if (!slabs.empty() && slabs[0].v.probe) {
      std::vector<unsigned long long> hp((size_t)sx::kProbeSlots * 16 * sx::kProbeEv);
      if (cudaMemcpy(hp.data(), slabs[0].v.probe, hp.size() * sizeof(hp[0]), cudaMemcpyDeviceToHost) == cudaSuccess)
        if (FILE* f = std::fopen(path, "wb")) {
          std::fwrite(hp.data(), sizeof(hp[0]), hp.size(), f);
          std::fclose(f);
        }
    }
  for (auto& g : seg)
    if (g) cudaGraphExecDestroy(g);
  for (auto& v : tev)
    for (auto e : v) cudaEventDestroy(e);
  for (void* p : ipc_open) cudaIpcCloseMemHandle(p);
  ipc_open.clear();
  if (comm) ncclCommDestroy(comm);
  for (void* p : allocs) cudaFree(p);
  allocs.clear();
  if (h_state) cudaFreeHost(h_state);
  if (h_err) cudaFreeHost(h_err);
  if (h_res) cudaFreeHost(h_res);
  if (h_slot) cudaFreeHost(h_slot);
  if (h_wcol) cudaFreeHost(h_wcol);
  if (ev_slot) cudaEventDestroy(ev_slot);
  for (auto q : xs)
    if (q) cudaStreamDestroy(q);
  for (auto e : ev_join)
    if (e) cudaEventDestroy(e);
  if (ev_fork) cudaEventDestroy(ev_fork);
  for (auto e : ev_done)
    if (e) cudaEventDestroy(e);
  if (ev_user) cudaEventDestroy(ev_user);
  if (ev_loop0) cudaEventDestroy(ev_loop0);
  if (ev_loop1) cudaEventDestroy(ev_loop1);
  if (stream) cudaStreamDestroy(stream);
}

// ====================================================================== C ABI
// Every call but destroy: a NULL handle is E_ARG; a handle latched after a fault in its device
// loop (exchange timeout, CUDA or NCCL error) is E_STATE — its device state is undefined.
#define HANDLE_OK(h)                                                                          \
  do {                                                                                        \
    if (!(h)) return fail(SIMPLEX_E_ARG, "NULL handle");                                      \
    if ((h)->faulted) return fail(SIMPLEX_E_STATE, "the handle faulted earlier; destroy it");  \
  } while (0)

extern "C" {

void simplex_default_options(simplex_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->struct_size = sizeof(simplex_options);
  o->tol_opt = 1e-7;
  o->tol_piv = 1e-10;
  o->max_pivots = 0;
  o->record_trace = 1;
  o->device = -1;
  o->nranks = 1;
  o->rank = 0;
  o->nccl_id = nullptr;
  o->stream = nullptr;
  o->virtual_ranks = 1;
  o->exchange = 0;
  o->segment_pivots = 0;
  o->time_kernels = 0;
  o->lookahead = 0;
  o->pivot_rule = 0;
  o->phase1 = 1;
  o->overlap = 1;
}

simplex_err simplex_create(simplex_t** out, int64_t m, int64_t n, const double* A, const double* b,
                           const double* c, const simplex_options* opt) {
  g_err.clear();
  if (!out) return fail(SIMPLEX_E_ARG, "out is NULL");
  *out = nullptr;
  if (m < 1 || n < 1) return fail(SIMPLEX_E_ARG, "m and n must be >= 1");
  if (!A || !b || !c) return fail(SIMPLEX_E_ARG, "NULL input pointer");
  simplex_options o;
  simplex_default_options(&o);
  if (opt) {
    if (opt->struct_size != sizeof(simplex_options)) return fail(SIMPLEX_E_ARG, "simplex_options.struct_size mismatch");
    o = *opt;
  }
  if (!(o.tol_opt >= 0.0) || !(o.tol_piv >= 0.0)) return fail(SIMPLEX_E_ARG, "tolerances must be >= 0");
  if (o.pivot_rule != 0 && o.pivot_rule != 1) return fail(SIMPLEX_E_ARG, "pivot_rule must be 0 (Dantzig) or 1 (Bland)");
  int prev = 0;
  cudaGetDevice(&prev);
  simplex_t* h = new simplex_s();
  simplex_err e = h->setup(m, n, b, &o);
  if (e == SIMPLEX_OK) e = h->load(A, b, c, true);
  cudaSetDevice(prev);
  if (e != SIMPLEX_OK) {
    std::string keep = g_err;
    h->release();
    delete h;
    g_err = keep;
    return e;
  }
  *out = h;
  return SIMPLEX_OK;
}

simplex_err simplex_reset(simplex_t* h, const double* A, const double* b, const double* c) {
  g_err.clear();
  HANDLE_OK(h);
  DeviceGuard dg(h->device);
  return h->load(A, b, c, false);
}

simplex_err simplex_iterate(simplex_t* h, int64_t max_pivots, int64_t* pivots_done, simplex_status* st) {
  g_err.clear();
  HANDLE_OK(h);
  DeviceGuard dg(h->device);
  long long done = 0;
  simplex_err e = h->run(max_pivots, &done);
  if (e == SIMPLEX_E_CUDA || e == SIMPLEX_E_NCCL) h->faulted = true;
  if (pivots_done) *pivots_done = done;
  if (st) *st = static_cast<simplex_status>(h->status);
  return e;
}

simplex_err simplex_solve(simplex_t* h, simplex_status* st) { return simplex_iterate(h, 0, nullptr, st); }

simplex_err simplex_get_solution(simplex_t* h, double* x, double* y, double* objective, int64_t* pivots,
                                 simplex_status* st) {
  g_err.clear();
  HANDLE_OK(h);
  DeviceGuard dg(h->device);
  RET(h->enter());
  RET(h->flush_all());
  CK(cudaMemsetAsync(h->d_x, 0, sizeof(double) * h->n, h->stream));
  CK(cudaMemsetAsync(h->d_y, 0, sizeof(double) * h->m, h->stream));
  for (int s = 0; s < h->nslabs; ++s)
    CK(sx::launch_extract(h->slabs[s].v, h->n, h->d_x, h->d_y, s == 0 ? h->d_obj : nullptr, h->stream));
  h->kernel_launches += h->nslabs;
  if (h->use_nccl()) NK(ncclAllReduce(h->d_y, h->d_y, (size_t)h->m, ncclFloat64, ncclSum, h->comm, h->stream));
  std::vector<double> hy;
  if (h->hybrid) {                          // the host lane's slack columns' entries of y
    hy.assign((size_t)h->m, 0.0);
    CK(cudaMemcpyAsync(hy.data(), h->d_y, sizeof(double) * h->m, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->lane.y_part(hy.data());
    CK(cudaMemcpyAsync(h->d_y, hy.data(), sizeof(double) * h->m, cudaMemcpyHostToDevice, h->stream));
  }
  if (x) CK(cudaMemcpyAsync(x, h->d_x, sizeof(double) * h->n, cudaMemcpyDefault, h->stream));
  if (y) CK(cudaMemcpyAsync(y, h->d_y, sizeof(double) * h->m, cudaMemcpyDefault, h->stream));
  double obj = 0.0;
  CK(cudaMemcpyAsync(&h->h_state[2].p, h->d_obj, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  obj = h->h_state[2].p;
  if (objective) *objective = obj;
  if (pivots) *pivots = h->it;
  if (st) *st = static_cast<simplex_status>(h->status);
  return SIMPLEX_OK;
}

simplex_err simplex_solve_lp(simplex_t* h, const double* A, const double* b, const double* c, double* x, double* y,
                             double* objective, int64_t* pivots, simplex_status* st) {
  g_err.clear();
  HANDLE_OK(h);
  if (!A || !b || !c) return fail(SIMPLEX_E_ARG, "NULL input pointer");
  if (!h->small) {                          // the three calls, in order (same results and errors)
    simplex_err e = simplex_reset(h, A, b, c);
    if (e == SIMPLEX_OK) e = simplex_solve(h, nullptr);
    if (e == SIMPLEX_OK) e = simplex_get_solution(h, x, y, objective, pivots, st);
    return e;
  }
  DeviceGuard dg(h->device);
  long long piv = 0;
  simplex_err e = h->solve_lp_small(A, b, c, x, y, objective, &piv);
  if (e == SIMPLEX_E_CUDA) h->faulted = true;
  if (pivots) *pivots = piv;
  if (st) *st = static_cast<simplex_status>(h->status);
  return e;
}

simplex_err simplex_get_trace(simplex_t* h, int32_t* k, int32_t* r, int64_t cap, int64_t* len) {
  g_err.clear();
  HANDLE_OK(h);
  DeviceGuard dg(h->device);
  const sx::SlabView& v = h->slabs[0].v;
  const long long n = std::min<long long>(std::min<long long>(h->it, v.trace_cap), std::max<int64_t>(cap, 0));
  if (n > 0) {
    if (!k || !r) return fail(SIMPLEX_E_ARG, "NULL trace buffer");
    CK(cudaMemcpyAsync(k, v.trace_k, sizeof(int32_t) * n, cudaMemcpyDefault, h->stream));
    CK(cudaMemcpyAsync(r, v.trace_r, sizeof(int32_t) * n, cudaMemcpyDefault, h->stream));
  }
  CK(cudaStreamSynchronize(h->stream));
  if (len) *len = n;
  return SIMPLEX_OK;
}

simplex_err simplex_get_tableau(simplex_t* h, double* T_out, int64_t ld_out) {
  g_err.clear();
  HANDLE_OK(h);
  if (!T_out) return fail(SIMPLEX_E_ARG, "NULL argument");
  DeviceGuard dg(h->device);
  long long cols = 1 + (h->hybrid ? h->lane.hw : 0);
  for (auto& sl : h->slabs) cols += sl.v.w;
  if (ld_out < cols) return fail(SIMPLEX_E_ARG, "ld_out smaller than the slab's logical columns");
  RET(h->enter());
  RET(h->flush_all());
  const long long base = h->slabs[0].v.c0;
  for (auto& sl : h->slabs) {
    const sx::SlabView& v = sl.v;
    CK(cudaMemcpy2DAsync(T_out + (v.c0 - base), sizeof(double) * ld_out, v.T, sizeof(double) * v.ld,
                         sizeof(double) * v.w, v.rows, cudaMemcpyDefault, h->stream));
  }
  if (h->hybrid)                                  // the host lane's columns
    CK(cudaMemcpy2DAsync(T_out + h->lane.c0, sizeof(double) * ld_out, h->lane.T.data(), sizeof(double) * h->lane.hw,
                         sizeof(double) * h->lane.hw, h->m + 1, cudaMemcpyDefault, h->stream));
  const sx::SlabView& v0 = h->slabs[0].v;
  CK(cudaMemcpy2DAsync(T_out + (cols - 1), sizeof(double) * ld_out, v0.T + v0.w, sizeof(double) * v0.ld,
                       sizeof(double), v0.rows, cudaMemcpyDefault, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return SIMPLEX_OK;
}

simplex_err simplex_tableau_hash(simplex_t* h, uint64_t* hash) {
  g_err.clear();
  HANDLE_OK(h);
  if (!hash) return fail(SIMPLEX_E_ARG, "NULL argument");
  DeviceGuard dg(h->device);
  RET(h->enter());
  CK(cudaMemsetAsync(h->d_hash, 0, sizeof(unsigned long long), h->stream));
  for (int s = 0; s < h->nslabs; ++s)
    CK(sx::launch_hash(h->slabs[s].v, h->W, (h->rank == 0 && s == 0) ? 1 : 0, h->d_hash, h->stream, h->sms));
  h->kernel_launches += h->nslabs;
  if (h->use_nccl())
    NK(ncclAllReduce(h->d_hash, h->d_hash, 1, ncclUint64, ncclSum, h->comm, h->stream));
  unsigned long long v = 0;
  CK(cudaMemcpyAsync(&h->h_state[2].it, h->d_hash, sizeof(v), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  std::memcpy(&v, &h->h_state[2].it, sizeof(v));
  if (h->hybrid) v += h->lane.hash();             // the host lane's columns (same formula, mod 2^64)
  *hash = v;
  return SIMPLEX_OK;
}

simplex_err simplex_get_stats(simplex_t* h, simplex_stats* s) {
  g_err.clear();
  if (!h || !s) return fail(SIMPLEX_E_ARG, "NULL argument");
  std::memset(s, 0, sizeof(*s));
  s->pivots = h->it;
  s->update_launches = h->upd_launches;
  s->update_ms_total = h->upd_ms;
  s->loop_ms_total = h->loop_ms;
  s->graph_launches = h->graph_launches;
  s->kernel_launches = h->kernel_launches;
  long long cols = 1 + (h->hybrid ? h->lane.hw : 0);
  for (auto& sl : h->slabs) cols += sl.v.w;
  s->local_rows = h->m + 1;
  s->local_cols = cols;
  s->local_ld = h->slabs[0].v.ld;
  s->col_offset = h->slabs[0].v.c0;
  s->bytes_per_pivot = 16LL * (h->m + 1) * cols;
  s->path = h->small ? 1 : h->hybrid ? 2 : (!h->slabs.empty() && h->slabs[0].v.look_nt > 0) ? 3 : 0;
  s->host_cols = h->hybrid ? h->lane.hw : 0;
  s->host_ms_total = h->host_ms;
  s->host_wait_ms_total = h->host_wait_ms;
  return SIMPLEX_OK;
}

simplex_err simplex_destroy(simplex_t* h) {
  if (!h) return SIMPLEX_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  h->release();
  delete h;
  cudaSetDevice(prev);
  return SIMPLEX_OK;
}

const char* simplex_last_error(void) { return g_err.c_str(); }

simplex_err simplex_nccl_unique_id(void* out128) {
  g_err.clear();
  if (!out128) return fail(SIMPLEX_E_ARG, "NULL output");
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return SIMPLEX_OK;
}

simplex_err simplex_partition(int64_t total_cols, int64_t nparts, int64_t part, int64_t* c0, int64_t* width) {
  if (total_cols < 1 || nparts < 1 || part < 0 || part >= nparts || !c0 || !width)
    return fail(SIMPLEX_E_ARG, "simplex_partition: bad arguments");
  // widths floor(total/P) or +1, the remainder to the lowest parts
  const int64_t base = total_cols / nparts, rem = total_cols % nparts;
  *c0 = part * base + std::min(part, rem);
  *width = base + (part < rem ? 1 : 0);
  return SIMPLEX_OK;
}

const char* simplex_version(void) { return "libsimplex 0.3.0 (sm_100a, dense full-tableau simplex)"; }

}  // extern "C"
