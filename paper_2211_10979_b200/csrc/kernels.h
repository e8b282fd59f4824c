// kernels.h — host-side launchers of the libsimplex kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

#include "device.cuh"

namespace sx {

// Experiment hooks (SIMPLEX_* environment variables used by scripts/ probes) exist only in
// builds compiled with -DSIMPLEX_EXPERIMENTS (build.build(defines=["SIMPLEX_EXPERIMENTS"],
// out=...)).  The product libsimplex.so never reads the environment: every behaviour of it
// is chosen by simplex_options.
inline const char* experiment_env(const char* name) {
#ifdef SIMPLEX_EXPERIMENTS
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

constexpr int kUpdateRows = 4;   // rows in flight per thread in k_update (measured)
constexpr int kUpdateCtasPerSm = 4;

cudaError_t launch_set_stop(DevState* st, long long stop_at, cudaStream_t s);
cudaError_t launch_build(const SlabView& s, const double* b, long long n, cudaStream_t st, int sms);
cudaError_t launch_init_state(const SlabView& s, long long n, long long cap, cudaStream_t st);
cudaError_t launch_price0(const SlabView& s, double tol_opt, cudaStream_t st);
cudaError_t launch_pack(const SlabView& s, double* send, int grid, cudaStream_t st, bool pdl);
cudaError_t launch_select(const SlabView& s, const XView& x, double tol_piv, int grid, cudaStream_t st,
                          bool pdl);
cudaError_t update_occupancy(int* blocks_per_sm);
cudaError_t launch_update(const SlabView& s, int q, double tol_opt, int grid, cudaStream_t st, bool pdl);
// k_lookahead: select up to S pivots into chain bank `bown`, chaining from T (bpre >= 0: first
// the pending pivots of bank bpre, whose pass runs concurrently)
// (cache: keep the previous bank's operands in shared memory when they fit)
constexpr size_t kLookCacheMax = 200 * 1024;
cudaError_t launch_lookahead(const SlabView& s, const double* T, int S, int bown, int bpre, double tol_opt,
                             double tol_piv, int cluster, bool cache, cudaStream_t st);
size_t lookahead_smem(const SlabView& s, int cluster, bool cache, int* nqc, int* nqr);
// k_look2 (the default single-part selection when its own-bank operands fit in shared memory):
// own column / row slots per thread and the dynamic shared memory (ps: previous bank too)
constexpr size_t kLook2SmemMax = 220 * 1024;
size_t look2_smem(const SlabView& s, int nt, bool ps, int qc, int qr);
// picks the k_look2 instantiation for the slab (s->look_*) and sets the kernel attributes; returns
// the hand-off size in double2 entries, 0 if k_look2 does not fit (the slab keeps k_lookahead)
long long look2_prepare(SlabView* s, int cluster);
// k_mlook: one pivot t (t = -1: block start) of the multi-part look-ahead, between two exchanges
// xp.n > 0: the slot goes to every rank's gather buffer over peer memory + flags (no NCCL)
cudaError_t launch_mlook(const SlabView& s, const double* xin, double* xout, int nparts, long long xstride, int t,
                         int S, double tol_opt, double tol_piv, int cluster, const XPeers& xp, cudaStream_t st);
// k_mblock: the whole block's multi-part selection in one launch (peer-memory exchange only)
// (T: the tableau the chains start from; bpre >= 0: the previous block's bank is chained first)
cudaError_t launch_mblock(const SlabView& s, const double* T, int nparts, long long xstride, int S, int bown,
                          int bpre, double tol_opt, double tol_piv, int cluster, const XPeers& xp, cudaStream_t st,
                          bool pdl = false);
int mblock_max_clusters(int cluster, int rows);
int lookahead_cluster_size();
int update_s_max(int S);
int pass_cfg_choice(bool pipelined, double pass_bytes);   // k_update_s configuration (R rows x K stages)
size_t update_s_smem(int cfg, int cw, int rows, int S);
cudaError_t update_s_occupancy(int cfg, int S, int* blocks_per_sm, size_t smem);
// k_update_s: apply the pivots of chain bank `bank` to src, writing dst (src == dst: in place)
cudaError_t launch_update_s(int cfg, const SlabView& s, int S, const double* src, double* dst, int bank, int nc,
                            int Gr, int cw, cudaStream_t st, bool pdl);
// k_solve_small: the whole solve of a tableau that fits in one CTA's shared memory, one launch
size_t small_smem_bytes(int rows, int w);
size_t small_smem_max();
// io.A != NULL (simplex_solve_lp): build Table I from device A, b, c in the kernel and write
// x, y and res = {objective, status, pivots, error bits} after the solve
cudaError_t launch_solve_small(const SlabView& s, long long stop_at, double tol_opt, double tol_piv,
                               cudaStream_t st, const SmallLP& io = SmallLP{});
cudaError_t launch_phase1_row0(const SlabView& s, cudaStream_t st);
cudaError_t launch_phase2_row0(const SlabView& s, long long n, cudaStream_t st);
// Phase I drive-out on the device (reading p4; kernels.cu k_drive_*)
cudaError_t launch_drive_find(const SlabView& s, int i, long long nm, double tol, long long* fj, cudaStream_t st);
cudaError_t launch_drive_pick(const long long* fj, int nparts, long long* fjmin, cudaStream_t st);
cudaError_t launch_drive_col(const SlabView& s, const long long* fjmin, double* xcol, cudaStream_t st);
cudaError_t launch_drive_force(const SlabView& s, int i, int q, const long long* fjmin, const double* xcols,
                               int nsrc, long long xs, cudaStream_t st);
cudaError_t launch_force(const SlabView& s, int r, int k, const double* col, cudaStream_t st);
cudaError_t launch_set_status(DevState* d, int status, cudaStream_t st);
cudaError_t launch_flush(const SlabView& s, cudaStream_t st);
cudaError_t launch_extract(const SlabView& s, long long n, double* x, double* y, double* obj, cudaStream_t st);
cudaError_t launch_hash(const SlabView& s, long long Wg, int include_rhs, unsigned long long* out,
                        cudaStream_t st, int sms);

}  // namespace sx
