// device.cuh — data structures shared by the libsimplex kernels and the host engine.
//
// Layout of one slab in HBM:
//   T        (m+1) x ld doubles, row-major, ld = roundup(w+1, 16) so every row starts on
//            a 128-byte line; local column j < w is global column c0 + j, local column w
//            is the (replicated) rhs "cv", columns w+1 .. ld-1 are zero
//            padding (they stay exactly zero: prow_j = 0/p = 0 and fma(-a, 0, 0) = 0).
//   col      m+1 (+2 pad) staged pivot column T[.][k]   (snapshot, read by the update)
//   rownorm  ld   normalized pivot row T[r][.]/p          (written back one pivot later)
//   price    nslot argmin candidates of the NEW row 0 per warp slot of 64 columns (fused pricing)
//   rcand    ratio-test block candidates
#pragma once
#include <cstdint>
#include <vector_types.h>

namespace sx {

constexpr int kRunning = -1;
constexpr int kOptimal = 0;
constexpr int kUnbounded = 2;
constexpr int kIterLimit = 4;

constexpr int kThreads = 256;              // threads per CTA for every kernel
constexpr int kMaxLook = 16;               // max pivots per look-ahead block (rank-s update)
constexpr int kLookThreads = 256;          // threads per CTA of the look-ahead selection (1 cluster)
constexpr int kColS = 2 * kMaxLook;        // colS row stride / prowS rows: two blocks (banks) of chains

constexpr uint32_t kErrNonFinite = 1u;
constexpr uint32_t kErrNegRhs = 2u;
constexpr uint32_t kErrExchange = 4u;      // peer-memory exchange timed out (status -> kFault)
constexpr int kFault = -2;                 // device loop stopped on an error (see err)

// (value, index) argmin candidate; "none" = (+inf, INT64_MAX).  Compared
// lexicographically, which equals the oracle's ascending strict-< scan when no NaN
// is present.
struct Cand {
  double v;
  long long idx;
};

// Device-resident loop state (one per slab).  Written only by the single "last
// block" of k_select (and by the host between launches); read by every kernel.
struct alignas(16) DevState {
  long long it;        // pivots done
  long long cap;       // iteration cap (reading c12)
  long long stop_at;   // stop before pivot number stop_at (simplex_iterate)
  double p;            // current pivot element T[r][k]
  int status;          // kRunning / kOptimal / kUnbounded / kIterLimit
  int go;              // 1: k_update must apply pivot (r, k, p)
  int r;               // pivot row, 1-based
  int k;               // entering column, global
  int pend_r;          // row whose normalized values still sit in rownorm (-1: none)
  unsigned int err;    // build/validation error bits
  unsigned int ticket; // last-block ticket of k_select
  unsigned int ticket2;
  int phase;           // 1: Phase I (artificials in the basis), 2: the problem's objective
  int drive_next;      // Phase I drive-out: index of the next listed row to drive out (reading p4)
  int pw;              // columns priced (local): all non-rhs in Phase I, no artificials after
  int sb[2];           // look-ahead: pivots selected into chain bank 0 / 1
  int rsb[2][kMaxLook];// look-ahead: their pivot rows, in order
  // pass timer (SlabView::time_pass): %globaltimer of the first CTA start / last CTA end of the
  // running k_update_s launch, CTAs finished, and the sum / count of launch durations
  unsigned long long pass_t0, pass_t1;
  unsigned int pass_done;
  long long pass_n;
  double pass_ns;
  // multi-part look-ahead over peer memory: exchanges this part has published (monotone over
  // the handle's life, never reset; every part counts the same)
  unsigned long long xseq;
};

// Destinations of a part's exchange slot in the peer-memory exchange of k_mlook.
// Every value travels as two 8-byte words {32 data bits, 32-bit sequence number} (the "LL"
// format: an aligned 8-byte store is single-copy atomic, so a reader that sees the expected
// sequence number in a word also sees that word's data) — no fence, no flag, no barrier: the
// writer stores its slot [v, k, col[0..m]] straight into buffer (t+1)&1 of EVERY rank's gather
// buffer (a peer's through its CUDA-IPC mapping, over NVLink) and each reader polls exactly the
// words it consumes.  Gather buffer: 2 parities x nparts slots x xstride values x 2 words.
constexpr int kMaxPeers = 8;
struct XPeers {
  int n;                               // destination ranks; 0 = exchange outside the kernel
  int part;                            // this part's slot index in every gather buffer
  long long half;                      // values per parity (nparts * xstride)
  unsigned long long* x[kMaxPeers];    // gather buffers of every rank (LL words)
  const unsigned long long* mine;      // this rank's gather buffer
  unsigned long long timeout_ns;       // a poll gives up after this long (options.exchange_timeout_ms)
};

struct SlabView {
  double* T;
  long long ld;
  int rows;            // m + 1
  int w;               // local non-rhs columns; rhs is local column w
  long long c0;        // global index of local column 0
  int rule;            // 0 Dantzig, 1 Bland (pivot_rule)
  int arts;            // artificial columns (rows with b_i < 0), global columns n+m .. n+m+arts-1
  int* art_of_row;     // [m] artificial index of row i+1, or -1
  int* neg_rows;       // [arts] rows (1-based) with b_i < 0, ascending
  double* cvec;        // [n] c, for the Phase II objective row
  int nslot;           // pricing slots: warps of 32 double2 of row 0 = ceil(ld/64)
  Cand* price;         // [nslot]
  double* col;         // [rows + 2]
  double* rownorm;     // [ld]
  Cand* rcand;         // [ratio-test blocks]
  int* basis;          // [m]
  int* trace_k;
  int* trace_r;
  long long trace_cap;
  DevState* st;
  // rank-s look-ahead (NEXT #1); NULL when the handle runs 1 pivot/pass.
  // Two banks of chains: bank q holds pivots u = 0..15 at colS[i][16q+u], prowS[16q+u][.]
  double* colS;        // [rows][kColS]     pivot columns T^t[.][k_t], t-minor
  double* prowS;       // [kColS][ld]       normalized pivot rows T^t[r_t][.] / p_t
  double* colT;        // [2][16][rows]     the same pivot columns, transposed (bank, t, row): the
                       //                   selection's per-row chain loads coalesce across a warp
  double* R0;          // [ld]              current objective row during selection
  double* RHS;         // [rows]            current rhs column during selection
  Cand* pcand;         // [look-ahead CTAs] Step-1 candidates per CTA
  // k_look2: hand-off of each launch's own-bank chain operands to the next launch
  // (2 banks x [own column slots q][8 pairs][G threads] + [own row slots][8][G], double2); NULL and
  // look_nt = 0: the selection is k_lookahead
  double2* hand;
  int look_nt;         // threads per CTA of k_look2 (0: k_lookahead)
  int look_qc, look_qr;     // k_look2 instantiation: own column / row slots per thread
  int look_nqc, look_nqr;   // own columns / rows per thread actually used (hand-off layout)
  unsigned long long* probe;   // experiment hook (SIMPLEX_PROBE): selection phase timestamps, else NULL
  int time_pass;       // 1: k_update_s times itself on the device (DevState pass_*) — the way to
                       // time the pipelined pass WHILE the selection runs next to it (event nodes
                       // between the two kernels would serialize them)
};

// k_lookahead phase timestamps (experiment hook): per launch slot (64), per CTA (16),
// kProbeEv %globaltimer stamps: start, after the first reduction, then per pivot t
// [phase A loads arrived, phase A done, CTA reduction A done, cluster barrier A done, reduction A
// done, phase B loads arrived, phase B done, CTA reduction B, cluster barrier B, reduction B done].
constexpr int kProbeSlots = 64;
constexpr int kProbeEv = 2 + 10 * kMaxLook;

// k_solve_small's LP mode (simplex_solve_lp): inputs (device pointers, A row-major m x n) and
// outputs (device: x [n], y [m], res = {objective, status, pivots, error bits}); A == NULL: off.
struct SmallLP {
  const double* A;
  const double* b;
  const double* c;
  long long n;
  double* x;
  double* y;
  double* res;
};

// Where k_select takes the entering column from.
struct XView {
  int nparts;          // parts (ranks x virtual slabs) the columns are split over
  const double* recv;  // NULL: entering column read from the own slab (one part);
                       // else nparts x stride gathered [v, k (int64 bits), col[0..m]]
  long long stride;
};

}  // namespace sx
