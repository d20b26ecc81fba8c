// Interface Krylov iteration of DDELM-NN on the device (sm_100a, fp64).
//
// cs_reduced_apply (solvers.cpp:372-386) with the theta-mixed Neumann-Neumann weight
// (solvers.cpp:599-603), in the reference's own grouping: K^+ is applied INTO coefficient space
// (c = K^+ phi, an M-vector) and the flux / Cdelta rows act on c afterwards
// (solvers.cpp:215-218, 240-241, 455, 468). With the factored pseudo-inverse K^+ = C Q_r^T
// (k_cod.cu) one operator application is, per subdomain i:
//   OP1   s = Q_G^T phi (+ Q_r^T f), corner parts t_i, psi_i = Zc v            (per subdomain)
//   OP2   mu|corners = Wmu [t; psi] ; c = C s - Ypi mu ; x_i = -F c            (streams C, F, Ypi)
//   NN1   y = Cbar (Qbar^T (-x|flux)) ; tr_i = Cdelta y                        (streams Cbar, Cdelta)
//   NN2   y = Cdelta^T tl ; zz_i = Qbar (Cbar^T y)                             (streams Cdelta, Cbar)
//   OP3   w = theta P^T P x + (1-theta) x ; u_i = C^T (F^T w)                  (streams F, C)
//   OP4   nu|corners = S^{-1} t' ; d2 rows ; o_i = -phi + Q_G(...) + Zc^T d2   (per subdomain)
//   XR    Ap = o gathered over the two owners of each Delta index ; x, r update (CG)
// The coarse solve mu = S^{-1}(t + Dpp^T psi) and d1 = psi - Dpp mu are applied through the
// precomputed rows Wmu = [S^{-1} | S^{-1} Dpp^T] and Wd = [-Dpp S^{-1} | I - Dpp S^{-1} Dpp^T]
// (k_blocks.cu), so every work item evaluates the handful of coarse rows it needs from the
// gathered [t; psi] vector itself: no single-CTA coarse phase, no extra grid barrier.
//
// HBM streaming (warp-specialised): in the four dense phases one work item is a row slice
// (rows j0..j1 of one subdomain's C, F, Cbar, Cdelta). Warp 15 is the producer: it walks the
// CTA's chunks and fills a 4-stage shared-memory ring with bulk copies on the TMA engine
// (cp.async.bulk, completion on a "full" mbarrier), refilling a stage once its "empty" mbarrier
// says all consumer warps released it. Warps 0..14 consume: each takes whole rows — a row-dot
// t_j = A_j . x against x held in registers, then the axpy y += t_j B_j into per-lane register
// accumulators — so there is no block barrier per chunk; the 15 warp partials are summed in a
// fixed order at the end of the item. The first chunks of the next phase are issued before the
// grid barrier (the matrices are constant during the solve), and NN2 / OP3 walk their slices in
// reverse so they start on the lines NN1 / OP2 left in L2.
//
// Two drivers share these phases. Default: OP1, ONE fused launch for OP2 -> NN1 -> NN2 -> OP3
// (kPhFused: between them an item waits only for its own and its edge neighbours' completion
// counters), OP4 and XR; the whole CG loop (solvers.cpp:82-119) captured as ONE CUDA graph with a
// device-side while node (the XR2 phase sets the loop condition). On a sharded workspace every
// phase is its own launch and the owner-slot exchanges sit between them. Alternative (DDELM_CG_MODE=persistent, one device): one persistent
// cooperative kernel with 7 grid barriers per iteration. In both, the CG scalars are sums of
// per-CTA / per-subdomain partials in a fixed order (no atomics: bitwise deterministic, and the two
// drivers agree bit for bit), the search direction is double-buffered so the p-update is fused
// into OP1, and the same phases apply the operator once (tests), form the reduced right-hand side
// (solvers.cpp:542-551) and reconstruct the coefficients (solvers.cpp:565-577).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "kernels.hpp"

namespace cgs = cooperative_groups;

namespace ddg {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kCWarps = kWarps - 1;  // consumer warps of a streamed phase
constexpr int kCThreads = kCWarps * 32;
constexpr int kProducerWarp = kWarps - 1;
constexpr int kStages = 4;
constexpr int kStageBytes = 32768;
constexpr int kMaxW = 1024;  // widest row-dot operand / axpy output (32 accumulators per lane)
constexpr int kRedW = 512;   // column chunk of the cross-warp accumulator reduction

/// Thread team of a phase: the whole CTA (512) or the consumer warps of a streamed phase (480,
/// named barrier 1 so the producer warp is never waited for).
struct Team {
  int n;
  __device__ __forceinline__ void sync() const {
    if (n == kThreads)
      __syncthreads();
    else
      asm volatile("bar.sync 1, %0;" ::"r"(kCThreads) : "memory");
  }
};
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, %0;" ::"r"(kCThreads) : "memory"); }

// ---------------------------------------------------------------- shared state of one CTA
struct Shared {
  double* ring;    // kStages x kStageBytes (also the Q_r^T staging area of OP1 / OP4)
  double* xa;      // row-dot operand (wmax)
  double* red;     // kCWarps x wred (warp partials of the axpy) / kThreads scratch
  double* z;       // [t; psi] (nz)
  double* t2;      // t' (n_pi)
  double* v1;      // per-subdomain vector (wmax)
  double* s0;      // rmax
  uint64_t* full;  // kStages
  uint64_t* empty; // kStages
  uint64_t* qbar;  // Q_r^T staging
};

__device__ __forceinline__ int wmax_of(const CgArgs& a) { return max(max(a.rmax, a.fmax), max(a.dmax, a.gmax)); }
__device__ __forceinline__ int wred_of(const CgArgs& a) {
  return min(kRedW, (max(max(a.rmax, a.fmax), a.dmax) + 31) & ~31);
}

__device__ __forceinline__ Shared carve(const CgArgs& a, uint64_t* bars) {
  extern __shared__ __align__(128) double smem[];
  Shared s;
  s.ring = smem;
  double* q = smem + kStages * (kStageBytes / 8);
  const int wm = wmax_of(a);
  s.xa = q;
  q += wm;
  s.red = q;
  q += max(kCWarps * wred_of(a), kThreads);
  s.z = q;
  q += a.n_pi + a.npf;
  s.t2 = q;
  q += max(a.n_pi, 1);
  s.v1 = q;
  q += wm;
  s.s0 = q;
  s.full = bars;
  s.empty = bars + kStages;
  s.qbar = bars + 2 * kStages;
  return s;
}

// ---------------------------------------------------------------- streamed phases
enum StreamKind { kOp2 = 0, kNn1 = 1, kNn2 = 2, kOp3 = 3 };

/// Geometry of one work item's stream: rows j0..j1 of a packed per-subdomain block (one bulk copy
/// per chunk). Row j holds A_j at column aoff, B_j at boff and (OP2) the 4 Ypi entries at yoff.
struct ItemGeo {
  const double* base;  // row j0 of the packed block
  int ld, aoff, boff, yoff, rows, wa, wb, rpc, nch;
  bool reverse;
};

__device__ __forceinline__ void part_rows(int rows, int P, int p, int& j0, int& j1) {
  const int chunk = (rows + P - 1) / P;
  j0 = min(rows, p * chunk);
  j1 = min(rows, j0 + chunk);
}

/// rows per chunk: a multiple of the consumer warp count when it fits a stage (one row per warp)
__host__ __device__ __forceinline__ int rows_per_chunk(int ld) {
  const int row = 8 * ld;
  const int k = kStageBytes / (kCWarps * row);
  return k > 0 ? min(k * kCWarps, 120) : max(1, kStageBytes / row);
}

__device__ __forceinline__ ItemGeo item_geo(const CgArgs& a, int kind, int i, int p, bool recon) {
  const SubGeo d = a.geo[i];
  const int R = a.rmax;
  const int ldf = d.kf_ld, ldd = d.kd_ld;
  ItemGeo g;
  if (a.compact && !recon) {
    // compact interface-level blocks (k_blocks.cu compact_stream_kernel): row q of KFc is
    // [e_q (rmax) | e_(q-r) (ncq) | (F [C Ypi])^T row q], row q of KDc is [e_q | (Cdelta Cbar)^T row q],
    // so the same row-dot / axpy machinery applies F C s - F Ypi mu (OP2), C^T F^T w (OP3), and
    // Cdelta Cbar v / Cbar^T Cdelta^T v (NN1 / NN2) without the M-long coefficient vector
    const int rows = kind == kOp2 ? d.r + a.ncq : (kind == kOp3 ? d.r : d.rb);
    int j0, j1;
    part_rows(rows, a.P, p, j0, j1);
    const double* KF = a.KFc + d.kfc_off + static_cast<size_t>(j0) * ldf;
    const double* KD = a.KDc + d.kdc_off + static_cast<size_t>(j0) * ldd;
    switch (kind) {
      case kOp2:  g = {KF, ldf, 0, R + a.ncq, R, j1 - j0, d.r, d.nF, 0, 0, false}; break;
      case kNn1:  g = {KD, ldd, 0, R, -1, j1 - j0, d.rb, d.nd, 0, 0, false}; break;
      case kNn2:  g = {KD, ldd, R, 0, -1, j1 - j0, d.nd, d.rb, 0, 0, true}; break;
      default:    g = {KF, ldf, R + a.ncq, 0, -1, j1 - j0, d.nF, d.r, 0, 0, true}; break;
    }
  } else {
    int j0, j1;
    part_rows(a.M, a.P, p, j0, j1);
    const double* KF = a.KF + d.kf_off + static_cast<size_t>(j0) * ldf;
    const double* KD = a.KD + d.kd_off + static_cast<size_t>(j0) * ldd;
    switch (kind) {
      case kOp2:  // A = C, Y = Ypi, B = F
        g = {KF, ldf, 0, recon ? -1 : R + a.ncq, R, j1 - j0, d.r, recon ? 0 : d.nF, 0, 0, false};
        break;
      case kNn1:  // A = Cbar, B = Cdelta
        g = {KD, ldd, 0, R, -1, j1 - j0, d.rb, d.nd, 0, 0, false};
        break;
      case kNn2:  // A = Cdelta, B = Cbar
        g = {KD, ldd, R, 0, -1, j1 - j0, d.nd, d.rb, 0, 0, true};
        break;
      default:    // OP3: A = F, B = C
        g = {KF, ldf, R + a.ncq, 0, -1, j1 - j0, d.nF, d.r, 0, 0, true};
        break;
    }
  }
  g.rpc = rows_per_chunk(g.ld);
  g.nch = (g.rows + g.rpc - 1) / g.rpc;
  return g;
}

__device__ __forceinline__ int n_items(int nwork) {
  const int b = blockIdx.x, G = gridDim.x;
  return b < nwork ? (nwork - 1 - b) / G + 1 : 0;
}
__device__ __forceinline__ bool reverse_kind(int kind) { return kind == kNn2 || kind == kOp3; }
/// item k of this CTA in traversal order; reverse phases walk items (and chunks) backwards
__device__ __forceinline__ int item_work(int k, int nitems, bool reverse) {
  return blockIdx.x + (reverse ? nitems - 1 - k : k) * gridDim.x;
}

/// Static data of a CTA's first work item of a streamed phase, loaded BEFORE griddepcontrol.wait
/// (it does not depend on the previous phase): the subdomain geometry, this thread's entry of the
/// phase's index table and (OP2) the coarse row of its corner. The prologue after the wait is
/// then one dependent load of fresh data instead of three.
struct StreamPre {
  int i;     // subdomain of the first item, -1: none
  int idx;   // OP3: fluxrow_delta, NN1 / NN2: ndelta_map, of row threadIdx.x (-1 beyond)
  int crow;  // OP2: Wmu row of corner threadIdx.x (threads < 4), -1 none
};
__device__ constexpr StreamPre kNoPre{-1, -1, -1};
/// the first item's geometry, shared by the CTA (kept out of registers across the wait)
__device__ __forceinline__ SubGeo& pre_geo() {
  __shared__ SubGeo g;
  return g;
}

__device__ __forceinline__ StreamPre stream_pre(const CgArgs& a, int kind) {
  StreamPre pre{-1, -1, -1};
  const int nitems = n_items(a.N * a.P);
  if (nitems == 0) return pre;
  const int w = item_work(0, nitems, kind == kNn2 || kind == kOp3);
  const int i = w / a.P;
  pre.i = i;
  if (threadIdx.x == 0) pre_geo() = a.geo[i];
  const int l = threadIdx.x;
  if (kind == kOp3) {
    if (l < a.fmax) pre.idx = a.fluxrow_delta[static_cast<size_t>(i) * a.fmax + l];
  } else if (kind == kNn1 || kind == kNn2) {
    if (l < a.dmax) pre.idx = a.ndelta_map[static_cast<size_t>(i) * a.dmax + l];
    // the Qbar_r^T rows of the prologue (NN1) / epilogue (NN2) GEMV: into L2 ahead of the wait
    const int E = a.ext;
    if (l < a.rmax) {
      const double* row = a.QtX + static_cast<size_t>(a.N + i) * a.rmax * E + static_cast<size_t>(l) * E;
      const unsigned long long lo = reinterpret_cast<unsigned long long>(row) & ~15ull;
      const unsigned long long hi = (reinterpret_cast<unsigned long long>(row + 1 + a.dmax) + 15ull) & ~15ull;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(static_cast<unsigned>(hi - lo)) : "memory");
    }
  } else if (kind == kOp2 && l < a.ncq && !a.one_level) {
    const int g = a.corner_q[i * a.ncq + l];
    pre.crow = g >= 0 ? a.gamma_pi[static_cast<size_t>(i) * a.gmax + g] : -1;
  }
  return pre;
}

/// Per-CTA timestamps of the streamed-phase trace (DDELM_CG_TRACE, phase-by-phase driver):
/// [0] kernel entry, [1] after griddepcontrol.wait, [2] first chunk consumed, [3] last chunk done,
/// [4] prologue done (consumers enter the stream).
__device__ __forceinline__ unsigned long long* phase_stamps() {
  __shared__ unsigned long long t[6];  // [5]: the item's gather done (first item)
  return t;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  return now;
}
/// trace of a per-subdomain phase (OP1 / OP4): slots s, s+1 = launch->wait, wait->end (CTAs with work)
__device__ __forceinline__ void trace_small(const CgArgs& a, int slot) {
  if (a.trace && threadIdx.x == 0 && blockIdx.x < a.N) {
    const unsigned long long* t = phase_stamps();
    double* tr = a.trace + blockIdx.x * 32 + slot;
    tr[0] += static_cast<double>(t[1] - t[0]);
    tr[1] += static_cast<double>(gtimer() - t[1]);
  }
}

/// Producer (warp 15, lane 0): walks the chunks of this CTA's items of one streamed phase.
/// `cnt` counts every chunk ever issued by this CTA: stage = cnt % kStages, use = cnt / kStages.
struct Producer {
  ItemGeo g;
  int kind, item, nitems, chunk;
  bool recon, active;
  unsigned cnt;
};

__device__ void producer_load_item(const CgArgs& a, Producer& pr) {
  if (pr.item < pr.nitems) {
    const int w = item_work(pr.item, pr.nitems, reverse_kind(pr.kind));
    pr.g = item_geo(a, pr.kind, w / a.P, w % a.P, pr.recon);
  }
}

__device__ void producer_begin(const CgArgs& a, Producer& pr, int kind, bool recon) {
  pr.kind = kind;
  pr.recon = recon;
  pr.nitems = n_items(a.N * a.P);
  pr.item = 0;
  pr.chunk = 0;
  pr.active = true;
  producer_load_item(a, pr);
}

/// Issue up to `limit` chunks (limit < 0: all remaining) of the current phase.
__device__ void producer_run(const CgArgs& a, Producer& pr, const Shared& sh, int limit) {
  while (pr.active && limit != 0) {
    while (pr.item < pr.nitems && pr.chunk >= pr.g.nch) {
      ++pr.item;
      pr.chunk = 0;
      producer_load_item(a, pr);
    }
    if (pr.item >= pr.nitems) {
      pr.active = false;
      break;
    }
    const ItemGeo& g = pr.g;
    const int c = g.reverse ? g.nch - 1 - pr.chunk : pr.chunk;
    const int ja = c * g.rpc, nr = min(g.rpc, g.rows - ja);
    const int st = pr.cnt % kStages;
    const unsigned use = pr.cnt / kStages;
    if (use > 0) mbar_wait(&sh.empty[st], (use - 1) & 1u);  // consumers released the stage
    double* dst = sh.ring + static_cast<size_t>(st) * (kStageBytes / 8);
    const uint32_t bytes = static_cast<uint32_t>(nr) * g.ld * 8;
    mbar_expect_tx(&sh.full[st], bytes);
    if (a.l2keep < 0) {
      bulk_g2s(dst, g.base + static_cast<size_t>(ja) * g.ld, bytes, &sh.full[st]);
    } else {
      // L2 reuse across phases: NN2 walks KD backwards right after NN1 walked it forwards, the next
      // OP2 walks KF forwards right after OP3 walked it backwards — the last l2keep/1000 of an NN1 /
      // OP3 item's walk stays in L2 (evict_last) for them; every other chunk streams evict_first
      const bool keep = (pr.kind == kNn1 || pr.kind == kOp3) && 1000 * (pr.chunk + 1) > (1000 - a.l2keep) * g.nch;
      const uint64_t pol = keep ? l2_policy_evict_last() : l2_policy_evict_first();
      bulk_g2s_hint(dst, g.base + static_cast<size_t>(ja) * g.ld, bytes, &sh.full[st], pol);
    }
    if (pr.kind == kNn2 && pr.chunk + 1 == g.nch && !a.compact) {
      // the item's epilogue reads Qbar_r^T (rb rows of the Kbar QtX block): into L2 while the last
      // chunks stream (the NN1-time prefetch has been evicted by the phase's own stream)
      const int w = item_work(pr.item, pr.nitems, true);
      const int i = w / a.P;
      const double* q0 = a.QtX + static_cast<size_t>(a.N + i) * a.rmax * a.ext;
      const unsigned long long lo = reinterpret_cast<unsigned long long>(q0) & ~15ull;
      const unsigned long long hi =
          (reinterpret_cast<unsigned long long>(q0 + static_cast<size_t>(a.rmax) * a.ext) + 15ull) & ~15ull;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(static_cast<unsigned>(hi - lo)) : "memory");
    }
    ++pr.chunk;
    ++pr.cnt;
    if (limit > 0) --limit;
  }
}

/// Prefetch into L2 the first |permille|/1000 (walk order) of this CTA's work items of a streamed
/// phase — issued while the HBM is idle (a latency-bound phase) so the phase later streams them from
/// L2. permille < 0: evict_last priority.
__device__ void l2_prefetch_items(const CgArgs& a, int kind, int permille) {
  const int nitems = n_items(a.N * a.P);
  const bool last = permille < 0;
  const int f = last ? -permille : permille;
  const uint64_t pol = l2_policy_evict_last();
  for (int k = 0; k < nitems; ++k) {
    const int w = item_work(k, nitems, reverse_kind(kind));
    const ItemGeo g = item_geo(a, kind, w / a.P, w % a.P, false);
    const int nr = static_cast<int>((static_cast<long long>(g.rows) * f) / 1000);
    if (nr <= 0) continue;
    const int r0 = g.reverse ? g.rows - nr : 0;
    unsigned long long lo = reinterpret_cast<unsigned long long>(g.base + static_cast<size_t>(r0) * g.ld) & ~15ull;
    const unsigned long long hi =
        (reinterpret_cast<unsigned long long>(g.base + static_cast<size_t>(r0 + nr) * g.ld) + 15ull) & ~15ull;
    constexpr unsigned long long kPiece = 1ull << 18;
    for (; lo < hi; lo += kPiece) {
      const unsigned sz = static_cast<unsigned>(min(kPiece, hi - lo));
      if (last)
        asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(lo), "r"(sz), "l"(pol)
                     : "memory");
      else
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(sz) : "memory");
    }
  }
}

/// L2 prefetch of the `n` chunks after the ones issued so far (this CTA's first item only): they
/// stream from HBM while the phase's prologue waits for fresh data, the ring being full.
__device__ void producer_l2ahead(const CgArgs& a, const Producer& pr, int n) {
  if (!pr.active || pr.item >= pr.nitems) return;
  const ItemGeo& g = pr.g;
  const int c0 = pr.chunk, c1 = min(g.nch, pr.chunk + n);
  if (c1 <= c0) return;
  // walk-order chunks c0 .. c1-1 are rows [ja, jb) (forward) or the mirrored range (reverse)
  int r0, r1;
  if (!g.reverse) {
    r0 = c0 * g.rpc;
    r1 = min(g.rows, c1 * g.rpc);
  } else {
    r1 = min(g.rows, (g.nch - c0) * g.rpc);
    r0 = (g.nch - c1) * g.rpc;
  }
  const unsigned long long lo = reinterpret_cast<unsigned long long>(g.base + static_cast<size_t>(r0) * g.ld) & ~15ull;
  const unsigned long long hi =
      (reinterpret_cast<unsigned long long>(g.base + static_cast<size_t>(r1) * g.ld) + 15ull) & ~15ull;
  if (hi > lo)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(static_cast<unsigned>(hi - lo)) : "memory");
}

/// Consumer side of one work item (warps 0..14): per row j of each chunk, t_j = A_j . xa
/// (xa in registers), u_j = hook(j, t_j, Ypi row) (lane-uniform), acc += u_j B_j (registers).
/// `ccnt` counts the chunks consumed by this CTA (mirrors the producer's cnt).
template <int W, class Hook>
__device__ void consume_item(const ItemGeo& g, const Shared& sh, unsigned& ccnt, double (&acc)[W], Hook hook,
                             bool tr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // W <= 16: the row-dot operand lives in registers; W = 32 (rows up to 1024 wide): it is read
  // from shared memory, the registers hold the 32 axpy accumulators
  constexpr bool kXs = W > 16;
  double xr[kXs ? 1 : W];
  // DDELM_CG_TRACE stamps (a %globaltimer read is not free: only when tracing)
  if (tr && threadIdx.x == 0 && phase_stamps()[4] == 0) phase_stamps()[4] = gtimer();
#pragma unroll
  for (int q = 0; q < W; ++q) {
    const int k = lane + 32 * q;
    if constexpr (!kXs) xr[q] = k < g.wa ? sh.xa[k] : 0.0;
    acc[q] = 0.0;
  }
  for (int cc = 0; cc < g.nch; ++cc) {
    const int c = g.reverse ? g.nch - 1 - cc : cc;
    const int ja = c * g.rpc, nr = min(g.rpc, g.rows - ja);
    const int st = ccnt % kStages;
    const double* S = sh.ring + static_cast<size_t>(st) * (kStageBytes / 8);
    mbar_wait(&sh.full[st], (ccnt / kStages) & 1u);
    if (tr && threadIdx.x == 0 && phase_stamps()[2] == 0) phase_stamps()[2] = gtimer();
    for (int rr = warp; rr < nr; rr += kCWarps) {
      const double* row = S + static_cast<size_t>(rr) * g.ld;
      const double* ar = row + g.aoff;
      double s = 0;
#pragma unroll
      for (int q = 0; q < W; ++q) {
        const int k = lane + 32 * q;
        if constexpr (kXs) {
          if (k < g.wa) s += ar[k] * sh.xa[k];
        } else {
          if (k < g.wa) s += ar[k] * xr[q];
        }
      }
      s = warp_sum(s);
      const double t = hook(ja + rr, s, row + g.yoff, lane);
      if (g.boff >= 0) {
        const double* br = row + g.boff;
#pragma unroll
        for (int q = 0; q < W; ++q) {
          const int l = lane + 32 * q;
          if (l < g.wb) acc[q] += br[l] * t;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.empty[st]);
    ++ccnt;
  }
  if (tr && threadIdx.x == 0) phase_stamps()[3] = gtimer();
}

/// Sum the consumer warps' accumulators (fixed warp order) and hand out column l values.
template <int W, class Out>
__device__ void reduce_warps(const CgArgs& a, const ItemGeo& g, const Shared& sh, const double (&acc)[W], Out out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wr = wred_of(a);
  for (int c0 = 0; c0 < g.wb; c0 += wr) {  // one chunk unless the rows are wider than kRedW
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int l = lane + 32 * q;
      if (l >= c0 && l < c0 + wr && l < g.wb) sh.red[warp * wr + (l - c0)] = acc[q];
    }
    cons_sync();
    const int nl = min(wr, g.wb - c0);
    for (int l = threadIdx.x; l < nl; l += kCThreads) {
      double s = 0;
      for (int w = 0; w < kCWarps; ++w) s += sh.red[w * wr + l];
      out(c0 + l, s);
    }
    cons_sync();
  }
}

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ double sum_parts(const double* base, size_t stride, int P, int idx) {
  // every part's load in flight before the (fixed-order) sum: the prologues are latency chains
  constexpr int kMaxP = 8;
  if (P <= kMaxP) {
    double v[kMaxP];
#pragma unroll
    for (int p = 0; p < kMaxP; ++p) v[p] = p < P ? __ldcg(base + p * stride + idx) : 0.0;
    double s = 0;
#pragma unroll
    for (int p = 0; p < kMaxP; ++p)
      if (p < P) s += v[p];
    return s;
  }
  double s = 0;
  for (int p = 0; p < P; ++p) s += __ldcg(base + p * stride + idx);
  return s;
}

/// sum over the two owner slots (each summed over the P parts) of Delta index g
__device__ __forceinline__ double gather_delta(const double* tab, const CgArgs& a, int g) {
  const size_t st = 2 * static_cast<size_t>(a.n_delta);
  return sum_parts(tab, st, a.P, 2 * g) + sum_parts(tab, st, a.P, 2 * g + 1);
}

__device__ __forceinline__ double gather_x(const CgArgs& a, int g) { return a.flip_sign[g] * gather_delta(a.xtab, a, g); }

/// one-level: dmu of cross flux row rr (= global flux row n_delta + rr), summed over its up to 4
/// owner slots and the P parts
__device__ __forceinline__ double gather_xc(const CgArgs& a, int rr) {
  const size_t st = 4 * static_cast<size_t>(a.npf);
  double s = 0;
  for (int k = 0; k < 4; ++k) s += sum_parts(a.xctab, st, a.P, rr * 4 + k);
  return a.flip_sign[a.n_delta + rr] * s;
}

/// z = [t; psi]: corner contributions of OP1 summed over their owners (subdomain order) and the
/// cross-flux data psi (mode 0: Dpd v; mode 1: dpi; mode 2: dpi - Dpd mu_Delta).
__device__ void gather_z(const CgArgs& a, const Shared& sh, int mode, int nthr) {
  // a thread's t and psi entries (fresh from OP1) are loaded together, then summed and stored:
  // one L2 round trip instead of two
  const int n = a.n_pi, nf = a.npf;
  for (int q = threadIdx.x; q < max(n, nf); q += nthr) {
    double t4[4] = {0, 0, 0, 0}, p4[4] = {0, 0, 0, 0}, dp = 0;
    if (q < n)
#pragma unroll
      for (int u = 0; u < 4; ++u) t4[u] = a.ttab[4 * static_cast<size_t>(q) + u];
    if (q < nf) {
      if (mode != 1)
#pragma unroll
        for (int u = 0; u < 4; ++u) p4[u] = a.ptab[4 * static_cast<size_t>(q) + u];
      if (mode != 0) dp = a.dpi[q];
    }
    if (q < n) sh.z[q] = ((t4[0] + t4[1]) + t4[2]) + t4[3];
    if (q < nf) {
      const double acc = (mode != 1) ? ((p4[0] + p4[1]) + p4[2]) + p4[3] : 0.0;
      sh.z[n + q] = (mode == 0) ? acc : (mode == 1 ? dp : dp - acc);
    }
  }
}

/// out[q] = W[row_q] . vec (len), one warp per row (warps < nwarps); rows < 0 give 0.
__device__ void rows_dot(const double* W, int ldw, const int* rows, int nrows, const double* vec, int len,
                         double* out, int nwarps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = warp; q < nrows; q += nwarps) {
    const int row = rows[q];
    double s = 0;
    if (row >= 0) {
      const double* w = W + static_cast<size_t>(row) * ldw;
      for (int k0 = lane; k0 < len; k0 += 256) {  // eight loads in flight per lane, summed in k order
        double wv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) wv[u] = k0 + 32 * u < len ? w[k0 + 32 * u] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (k0 + 32 * u < len) s += wv[u] * vec[k0 + 32 * u];
      }
    }
    s = warp_sum(s);
    if (lane == 0) out[q] = s;
  }
}

/// Deterministic sum of n values: lanes stride the array, then the xor tree (bitwise identical in
/// every lane, warp and CTA).
__device__ __forceinline__ double det_sum(const double* p, int n) {
  // the values are fresh (written by other CTAs / the previous phase): all of a lane's loads go out
  // before its (unchanged, in-order) sum — one L2 round trip per 8 values instead of one per value
  constexpr int kB = 8;
  double s = 0;
  for (int k0 = threadIdx.x & 31; k0 < n; k0 += 32 * kB) {
    double v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) v[u] = k0 + 32 * u < n ? p[k0 + 32 * u] : 0.0;
#pragma unroll
    for (int u = 0; u < kB; ++u)
      if (k0 + 32 * u < n) s += v[u];
  }
  return warp_sum(s);
}

/// y[k] = sum_e Q[k*ldq + e] x[e] for k < nk, e < ne: a warp per 4 rows (warps < nwarps).
__device__ void rowdot4(const double* Q, int ldq, int nk, int ne, const double* x, double* y, int nwarps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k0 = 4 * warp; k0 < nk; k0 += 4 * nwarps) {
    double c[4] = {0, 0, 0, 0};
    int e = lane;
    for (; e + 32 < ne; e += 64) {  // 8 loads in flight per lane (latency-bound prologues)
      double q0[4], q1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double* qr = Q + static_cast<size_t>(k0 + u < nk ? k0 + u : k0) * ldq;
        q0[u] = qr[e];
        q1[u] = qr[e + 32];
      }
      const double x0 = x[e], x1 = x[e + 32];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] += q0[u] * x0;
        c[u] += q1[u] * x1;
      }
    }
    for (; e < ne; e += 32) {
      const double xe = x[e];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k0 + u < nk) c[u] += Q[static_cast<size_t>(k0 + u) * ldq + e] * xe;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double v = warp_sum(c[u]);
      if (lane == 0 && k0 + u < nk) y[k0 + u] = v;
    }
  }
}

/// y[k] = sum_e Q[k*ldq + e] x[e] for k < nk, e < ne: each warp takes blocks of up to 8
/// consecutive rows (ceil(nk / nwarps) <= 8: one block per warp) and issues all of a batch's
/// loads (8 rows x 4 columns per lane) before its FMAs — one memory latency per 128 columns
/// instead of one per 32 (latency-bound prologues).
__device__ void rowdot_wide(const double* Q, int ldq, int nk, int ne, const double* x, double* y, int nwarps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= nwarps) return;
  const int rpw = min(8, (nk + nwarps - 1) / nwarps);
  constexpr int kE = 4;
  for (int k0 = warp * rpw; k0 < nk; k0 += nwarps * rpw) {
    double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int e0 = lane; e0 < ne; e0 += 32 * kE) {
      double q[8][kE];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int t = 0; t < kE; ++t) {
          const int e = e0 + 32 * t;
          q[u][t] = (u < rpw && k0 + u < nk && e < ne) ? Q[static_cast<size_t>(k0 + u) * ldq + e] : 0.0;
        }
#pragma unroll
      for (int t = 0; t < kE; ++t) {
        const int e = e0 + 32 * t;
        const double xe = e < ne ? x[e] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] += q[u][t] * xe;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double v = warp_sum(c[u]);
      if (lane == 0 && u < rpw && k0 + u < nk) y[k0 + u] = v;
    }
  }
}

/// y[c] = sum_k Q[k*ldq + c] x[k] for c < nc (<= team size), k < nk: threads over (c, k-group),
/// the k-groups combined in a fixed order through red (>= team size doubles).
template <class Out>
__device__ void coldot_split(const double* Q, int ldq, int nk, int nc, const double* x, double* red, Team tm,
                             Out out) {
  const int ncp = max(32, (nc + 31) & ~31);
  const int G = max(1, tm.n / ncp);
  const int c = threadIdx.x % ncp, grp = threadIdx.x / ncp;
  double s = 0;
  if (grp < G && c < nc) {
    const int k0 = (nk * grp) / G, k1 = (nk * (grp + 1)) / G;
    double s1 = 0;
    int k = k0;
    for (; k + 11 < k1; k += 12) {  // twelve loads in flight
      double q[12];
#pragma unroll
      for (int u = 0; u < 12; ++u) q[u] = Q[static_cast<size_t>(k + u) * ldq + c];
#pragma unroll
      for (int u = 0; u < 12; u += 2) {
        s += q[u] * x[k + u];
        s1 += q[u + 1] * x[k + u + 1];
      }
    }
    for (; k + 3 < k1; k += 4) {  // four loads in flight
      const double q0 = Q[static_cast<size_t>(k) * ldq + c], q1 = Q[static_cast<size_t>(k + 1) * ldq + c];
      const double q2 = Q[static_cast<size_t>(k + 2) * ldq + c], q3 = Q[static_cast<size_t>(k + 3) * ldq + c];
      s += q0 * x[k];
      s1 += q1 * x[k + 1];
      s += q2 * x[k + 2];
      s1 += q3 * x[k + 3];
    }
    for (; k + 1 < k1; k += 2) {
      s += Q[static_cast<size_t>(k) * ldq + c] * x[k];
      s1 += Q[static_cast<size_t>(k + 1) * ldq + c] * x[k + 1];
    }
    if (k < k1) s += Q[static_cast<size_t>(k) * ldq + c] * x[k];
    s += s1;
  }
  if (threadIdx.x < tm.n) red[threadIdx.x] = s;
  tm.sync();
  if (grp == 0 && c < nc) {
    double t = 0;
    for (int q = 0; q < G; ++q) t += red[q * ncp + c];
    out(c, t);
  }
  tm.sync();
}

/// Q_r^T [f E] rows (k < r) of local matrix t staged into the (idle) ring with one bulk copy;
/// falls back to the global copy when it does not fit. `cached` remembers what the ring holds.
struct QtxStage {
  unsigned cnt;
  int cached;
  bool pending;  // a bulk copy into the ring is in flight for `cached`
};

/// Staged per-subdomain blocks of OP1 / OP4: Q_r^T [f | E] rows k < r (ldq = ext) and Zc.
struct Staged {
  const double* qtx;
  const double* zc;
};

/// Issue the bulk copies of subdomain i's Q_r^T / Zc into the (idle) ring; false if they do not fit.
__device__ bool stage_issue(const CgArgs& a, const Shared& sh, QtxStage& q, int i, int r, size_t* qbytes) {
  const double* src = a.QtX + static_cast<size_t>(i) * a.rmax * a.ext;
  const double* zsrc = a.Zc + static_cast<size_t>(i) * a.crmax * a.gmax;
  const int rows = min(a.rmax, (r + 1) & ~1);
  const size_t bytes = static_cast<size_t>(rows) * a.ext * 8;
  const size_t zbytes = (static_cast<size_t>(a.crmax) * a.gmax * 8 + 15) / 16 * 16;  // Zc has 16 B of tail padding
  *qbytes = bytes;
  if (rows == 0 || bytes + zbytes > static_cast<size_t>(kStages) * kStageBytes) return false;
  if (threadIdx.x == 0) {
    mbar_expect_tx(sh.qbar, static_cast<uint32_t>(bytes + zbytes));
    bulk_g2s(sh.ring, src, static_cast<uint32_t>(bytes), sh.qbar);
    bulk_g2s(sh.ring + bytes / 8, zsrc, static_cast<uint32_t>(zbytes), sh.qbar);
  }
  q.cached = i;
  q.pending = true;
  return true;
}

__device__ Staged stage_qtx(const CgArgs& a, const Shared& sh, QtxStage& q, int i, int r) {
  const double* src = a.QtX + static_cast<size_t>(i) * a.rmax * a.ext;
  const double* zsrc = a.Zc + static_cast<size_t>(i) * a.crmax * a.gmax;
  size_t bytes = 0;
  if (q.cached != i) {
    __syncthreads();  // previous readers of the ring are done
    if (!stage_issue(a, sh, q, i, r, &bytes)) return {src, zsrc};
  } else {
    const int rows = min(a.rmax, (r + 1) & ~1);
    bytes = static_cast<size_t>(rows) * a.ext * 8;
  }
  if (q.pending) {
    mbar_wait(sh.qbar, q.cnt & 1u);
    ++q.cnt;
    q.pending = false;
  }
  return {sh.ring, sh.ring + bytes / 8};
}

/// Up to 32 independent row dots (one warp each): out[q] = W_q[row_q] . vec_q (rows < 0 give 0).
struct RowTask {
  const double* W;
  const double* vec;
  double* out;
  int ld, row, len;
};

__device__ void row_tasks(const RowTask* tk, int ntask, int nwarps) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = warp; q < ntask; q += nwarps) {
    const RowTask t = tk[q];
    double s = 0;
    if (t.row >= 0) {
      const double* w = t.W + static_cast<size_t>(t.row) * t.ld;
      for (int k0 = lane; k0 < t.len; k0 += 256) {  // eight loads in flight per lane, summed in k order
        double wv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) wv[u] = k0 + 32 * u < t.len ? w[k0 + 32 * u] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (k0 + 32 * u < t.len) s += wv[u] * t.vec[k0 + 32 * u];
      }
    }
    s = warp_sum(s);
    if (lane == 0) *t.out = s;
  }
}

// ---------------------------------------------------------------- OP1 (per subdomain, all warps)
/// mode 0: operator on v (CG: v = r + beta p_cur, written to p_next by the first owner);
/// mode 1: reduced right-hand side (phi = 0, + Q_r^T f); mode 2: reconstruction (phi = +v).
__device__ void dev_op1(const CgArgs& a, const Shared& sh, QtxStage& qs, int i, const double* v, int mode,
                        bool cg, double beta, const double* pcur, double* pnext) {
  const SubGeo d = a.geo[i];
  const int r = d.r, R = a.rmax, E = a.ext;
  double* vg = sh.v1;
  double* phi = sh.red;  // n_gamma <= kThreads (checked on the host)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int* gd = a.gamma_delta + static_cast<size_t>(i) * a.gmax;
  const int* gpi = a.gamma_pi + static_cast<size_t>(i) * a.gmax;
  for (int g = threadIdx.x; g < d.n_gamma; g += kThreads) {
    int dg = gd[g];
    if (dg < 0 && a.one_level && gpi[g] >= 0) dg = a.n_delta + gpi[g];  // mu_Pi entry (apply_B)
    double vv = 0.0;
    if (dg >= 0 && mode != 1) {
      if (cg) {
        // p_next = r + beta p_cur (solvers.cpp:116), the same rounding as XR1's replicated update;
        // every local owner stores it for OP4 (a sharded rank may hold only the second owner)
        vv = __fma_rn(beta, pcur[dg], a.r[dg]);
        if (dg < a.n_delta) pnext[dg] = vv;
      } else {
        vv = v[dg];
      }
    }
    vg[g] = vv;
    phi[g] = (mode == 0) ? -vv : vv;
  }
  const Staged stg = stage_qtx(a, sh, qs, i, r);
  const double* QtX = stg.qtx;
  __syncthreads();
  if (mode != 1) {
    rowdot4(QtX + 1, E, r, d.n_gamma, phi, sh.s0, kWarps);
  } else {
    for (int k = threadIdx.x; k < r; k += kThreads) sh.s0[k] = 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < r; k += kThreads) {
    double acc = sh.s0[k];
    if (mode >= 1) acc += QtX[static_cast<size_t>(k) * E];
    sh.s0[k] = acc;
    a.s[static_cast<size_t>(i) * R + k] = acc;
  }
  __syncthreads();
  if (a.one_level) {
    // no coarse space; the first owner of each corner writes the Pi entries of p_next
    if (cg && threadIdx.x < a.ncq) {
      const int g = a.corner_q[i * a.ncq + threadIdx.x];
      const int dst = a.corner_dst[i * a.ncq + threadIdx.x];
      if (g >= 0 && dst >= 0) pnext[a.n_delta + gpi[g]] = vg[g];
    }
  } else if (warp < a.ncq) {
    const int g = a.corner_q[i * a.ncq + warp];
    double acc = 0;
    if (g >= 0)
      for (int k = lane; k < r; k += 32) acc += QtX[static_cast<size_t>(k) * E + 1 + g] * sh.s0[k];
    acc = warp_sum(acc);
    const int dst = a.corner_dst[i * a.ncq + warp];
    if (lane == 0 && dst >= 0) a.ttab_w[dst] = acc;  // t(gp) -= phi - Ky at the corners (phi = 0 there)
  } else if (mode != 1) {
    // psi_i = Zc v (Dpd rows restricted to this subdomain), warps ncq..
    const double* Zc = stg.zc;
    for (int rho = warp - a.ncq; rho < a.crmax; rho += kWarps - a.ncq) {
      double acc = 0;
      for (int g = lane; g < d.n_gamma; g += 32) acc += Zc[static_cast<size_t>(rho) * a.gmax + g] * vg[g];
      acc = warp_sum(acc);
      const int dst = a.cross_dst[static_cast<size_t>(i) * a.crmax + rho];
      if (lane == 0 && dst >= 0) a.ptab_w[dst] = acc;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- streamed phases (consumers)
template <int W>
__device__ void dev_op2(const CgArgs& a, const Shared& sh, unsigned& ccnt, int mode, const StreamPre& pre) {
  const int nitems = n_items(a.N * a.P);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double muc[kMaxCq];
  __shared__ int crow[kMaxCq];
  for (int k = 0; k < nitems; ++k) {
    const int w = item_work(k, nitems, false);
    const int i = w / a.P, p = w % a.P;
    const bool first = (k == 0 && pre.i == i);
    // s_i (fresh from OP1) is loaded together with gather_z's t / psi slots: one round trip
    const int r = first ? pre_geo().r : a.geo[i].r;
    const double s_first = threadIdx.x < r ? a.s[static_cast<size_t>(i) * a.rmax + threadIdx.x] : 0.0;
    if (!a.one_level) gather_z(a, sh, mode, kCThreads);
    if (threadIdx.x < a.ncq) {
      if (first) {
        crow[threadIdx.x] = pre.crow;
      } else {
        const int g = a.corner_q[i * a.ncq + threadIdx.x];
        crow[threadIdx.x] = (g >= 0 && !a.one_level) ? a.gamma_pi[static_cast<size_t>(i) * a.gmax + g] : -1;
      }
    }
    for (int kk = threadIdx.x; kk < r; kk += kCThreads)
      sh.xa[kk] = kk == threadIdx.x ? s_first : a.s[static_cast<size_t>(i) * a.rmax + kk];
    cons_sync();
    const int nz = a.n_pi + a.npf;
    rows_dot(a.Wmu, nz, crow, a.ncq, sh.z, nz, muc, kCWarps);  // mu = S^{-1}(t + Dpp^T psi); 0 one-level
    if (mode == 2 && w == 0 && !a.one_level)  // mu_Pi of the solution (one CTA writes it)
      for (int gp = warp; gp < a.n_pi; gp += kCWarps) {
        double s = 0;
        const double* wr = a.Wmu + static_cast<size_t>(gp) * nz;
        for (int kk = lane; kk < nz; kk += 32) s += wr[kk] * sh.z[kk];
        s = warp_sum(s);
        if (lane == 0) a.mu_pi_out[gp] = s;
      }
    cons_sync();
    const ItemGeo g = item_geo(a, kOp2, i, p, mode == 2);
    int j0, j1;
    part_rows(a.M, a.P, p, j0, j1);
    double* coef = a.coeffs + static_cast<size_t>(i) * a.M;
    const double m0 = muc[0], m1 = muc[1], m2 = muc[2], m3 = muc[3];
    const int ncq = a.ncq;
    double acc[W];
    // reference grouping (solvers.cpp:336, 342): c = K^+ phi - Ypi mu, then F c
    const bool one = a.one_level != 0;
    consume_item<W>(g, sh, ccnt, acc, [&](int jr, double cs, const double* y, int ln) {
      double ym = ((y[0] * m0 + y[1] * m1) + y[2] * m2) + y[3] * m3;
      for (int q = 4; q < ncq; ++q) ym += y[q] * muc[q];  // biharmonic: second-component corners
      const double cj = one ? cs : cs - ym;
      if (mode == 2 && ln == 0) coef[j0 + jr] = cj;
      return cj;
    }, a.trace != nullptr);
    if (mode == 2) continue;
    double* xt = a.xtab_w + static_cast<size_t>(p) * 2 * a.n_delta;
    const int* fdst = a.flux_dst + static_cast<size_t>(i) * a.fmax;
    reduce_warps<W>(a, g, sh, acc, [&](int l, double s) {
      const int dst = fdst[l];
      if (dst >= 0) xt[dst] = -s;
      if (one) sh.v1[l] = s;
    });
    if (one) {
      // cross flux rows (apply_A, solvers.cpp:209-224): this subdomain's weighted share of every
      // cross row it touches (mean_edge: 1/(n-1) over the edge's points), one warp per row
      cons_sync();
      const int* off = a.cr_off + static_cast<size_t>(i) * (a.crmax + 1);
      double* xc = a.xctab_w + static_cast<size_t>(p) * 4 * a.npf;
      for (int rho = warp; rho < a.crmax; rho += kCWarps) {
        const int dst = a.cross_dst[static_cast<size_t>(i) * a.crmax + rho];
        if (dst < 0) continue;
        double v = 0;
        for (int e = off[rho] + lane; e < off[rho + 1]; e += 32) v += a.cr_w[e] * sh.v1[a.cr_l[e]];
        v = warp_sum(v);
        if (lane == 0) xc[dst] = -v;
      }
      cons_sync();
    }
  }
}

template <int W>
__device__ void dev_nn1(const CgArgs& a, const Shared& sh, unsigned& ccnt, const StreamPre& pre) {
  const int nitems = n_items(a.N * a.P);
  for (int k = 0; k < nitems; ++k) {
    const int w = item_work(k, nitems, false);
    const int i = w / a.P, p = w % a.P;
    const bool first = (k == 0 && pre.i == i);
    const SubGeo d = first ? pre_geo() : a.geo[i];
    const int nd = d.nd, rb = d.rb, E = a.ext;
    const double* QtX = a.QtX + static_cast<size_t>(a.N + i) * a.rmax * E;
    const int* nmap = a.ndelta_map + static_cast<size_t>(i) * a.dmax;
    for (int kk = threadIdx.x; kk < nd; kk += kCThreads)
      sh.v1[kk] = -gather_x(a, (first && kk == threadIdx.x) ? pre.idx : nmap[kk]);
    cons_sync();
    if (a.trace && threadIdx.x == 0 && phase_stamps()[5] == 0) phase_stamps()[5] = gtimer();
    rowdot_wide(QtX + 1, E, rb, nd, sh.v1, sh.xa, kCWarps);  // Qbar_r^T rhs (rhs nonzero on flux rows only)
    cons_sync();
    const ItemGeo g = item_geo(a, kNn1, i, p, false);
    double acc[W];
    // reference order (solvers.cpp:455): y = Kbar^+ rhs (M-vector), then Cdelta y
    consume_item<W>(g, sh, ccnt, acc, [](int, double cs, const double*, int) { return cs; }, a.trace != nullptr);
    double* trt = a.trtab_w + static_cast<size_t>(p) * 2 * a.n_delta;
    const int* ndst = a.nd_dst + static_cast<size_t>(i) * a.dmax;
    reduce_warps<W>(a, g, sh, acc, [&](int l, double s) { trt[ndst[l]] = s; });
  }
}

template <int W>
__device__ void dev_nn2(const CgArgs& a, const Shared& sh, unsigned& ccnt, const StreamPre& pre) {
  const int nitems = n_items(a.N * a.P);
  for (int k = 0; k < nitems; ++k) {
    const int w = item_work(k, nitems, true);
    const int i = w / a.P, p = w % a.P;
    const bool first = (k == 0 && pre.i == i);
    const SubGeo d = first ? pre_geo() : a.geo[i];
    const int nd = d.nd, rb = d.rb, E = a.ext;
    const double* QtX = a.QtX + static_cast<size_t>(a.N + i) * a.rmax * E;
    const int* nmap = a.ndelta_map + static_cast<size_t>(i) * a.dmax;
    const size_t st = static_cast<size_t>(a.N) * a.dmax;
    for (int kk = threadIdx.x; kk < nd; kk += kCThreads) {
      const int gg = (first && kk == threadIdx.x) ? pre.idx : nmap[kk];
      sh.xa[kk] = gather_delta(a.trtab, a, gg);
    }
    cons_sync();
    const ItemGeo g = item_geo(a, kNn2, i, p, false);
    double acc[W];
    // reference order (solvers.cpp:468): x = Cdelta^T tl (M-vector), then (Kbar^+)^T x
    consume_item<W>(g, sh, ccnt, acc, [](int, double cs, const double*, int) { return cs; }, a.trace != nullptr);
    reduce_warps<W>(a, g, sh, acc, [&](int l, double s) { sh.s0[l] = s; });
    // zz = Qbar_r (Cbar^T x) on the flux rows (partial over the parts p; linear)
    double* zzt = a.zztab_w + static_cast<size_t>(p) * 2 * a.n_delta;
    const int* ndst = a.nd_dst + static_cast<size_t>(i) * a.dmax;
    coldot_split(QtX + 1, E, rb, nd, sh.s0, sh.red, Team{kCThreads}, [&](int kk, double v) { zzt[ndst[kk]] = v; });
  }
}

template <int W>
__device__ void dev_op3(const CgArgs& a, const Shared& sh, unsigned& ccnt, const StreamPre& pre) {
  const int nitems = n_items(a.N * a.P);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < nitems; ++k) {
    const int w = item_work(k, nitems, true);
    const int i = w / a.P, p = w % a.P;
    const bool first = (k == 0 && pre.i == i);
    const SubGeo d = first ? pre_geo() : a.geo[i];
    const int r = d.r, R = a.rmax, E = a.ext;
    const double* QtX = a.QtX + static_cast<size_t>(i) * R * E;
    const int* fd = a.fluxrow_delta + static_cast<size_t>(i) * a.fmax;
    const double theta = a.theta;
    const size_t st = static_cast<size_t>(a.N) * a.dmax;
    for (int l = threadIdx.x; l < d.nF; l += kCThreads) {
      const int gg = (first && l == threadIdx.x) ? pre.idx : fd[l];
      double wv = 0.0;
      if (gg >= 0) {
        // every load of both gathers issued before any sum: a line the previous phase wrote costs
        // ~2 us on first touch (cross-die L2), so one round trip, not one per gather; the sums keep
        // gather_delta's order (bitwise unchanged)
        double zz = 0.0, x = 0.0;
        constexpr int kQ = 4;
        if (a.P <= kQ) {
          const size_t st2 = 2 * static_cast<size_t>(a.n_delta);
          double zv[2][kQ], xv[2][kQ];
#pragma unroll
          for (int sl = 0; sl < 2; ++sl)
#pragma unroll
            for (int pp = 0; pp < kQ; ++pp) {
              const size_t o = pp * st2 + 2 * static_cast<size_t>(gg) + sl;
              zv[sl][pp] = (pp < a.P && a.use_neumann) ? __ldcg(a.zztab + o) : 0.0;
              xv[sl][pp] = pp < a.P ? __ldcg(a.xtab + o) : 0.0;
            }
          const double fs = a.flip_sign[gg];
          double z0 = 0, z1 = 0, x0 = 0, x1 = 0;
#pragma unroll
          for (int pp = 0; pp < kQ; ++pp)
            if (pp < a.P) {
              z0 += zv[0][pp];
              z1 += zv[1][pp];
              x0 += xv[0][pp];
              x1 += xv[1][pp];
            }
          zz = z0 + z1;
          x = fs * (x0 + x1);
        } else {
          if (a.use_neumann) zz = gather_delta(a.zztab, a, gg);
          x = gather_x(a, gg);
        }
        if (a.use_neumann) {
          const double ptp = -zz;
          wv = theta * ptp;
          if (theta < 1.0) wv += (1.0 - theta) * x;
        } else {
          wv = x;
        }
      }
      sh.xa[l] = wv;  // apply_AT_delta: a(lrow) = w(grow) on the Delta flux rows
    }
    if (a.trace) {
      cons_sync();
      if (threadIdx.x == 0 && phase_stamps()[5] == 0) phase_stamps()[5] = gtimer();
    }
    if (a.one_level) {
      // apply_AT over the cross rows too (solvers.cpp:230-244): a(lrow) += w dmu(cross row)
      const int* off = a.cr_off + static_cast<size_t>(i) * (a.crmax + 1);
      const int* crr = a.cr_row + static_cast<size_t>(i) * a.crmax;
      for (int rho = threadIdx.x; rho < a.crmax; rho += kCThreads) sh.z[rho] = crr[rho] >= 0 ? gather_xc(a, crr[rho]) : 0.0;
      cons_sync();
      for (int l = threadIdx.x; l < d.nF; l += kCThreads) {
        double add = 0;
        for (int rho = 0; rho < a.crmax; ++rho) {
          if (crr[rho] < 0) continue;
          for (int e = off[rho]; e < off[rho + 1]; ++e)
            if (a.cr_l[e] == l) add += a.cr_w[e] * sh.z[rho];
        }
        sh.xa[l] += add;
      }
    }
    cons_sync();
    const ItemGeo g = item_geo(a, kOp3, i, p, false);
    double acc[W];
    // reference order: at = F^T a (M-vector, apply_AT), then (K^+)^T at = Q_r (C^T at)
    consume_item<W>(g, sh, ccnt, acc, [](int, double cs, const double*, int) { return cs; }, a.trace != nullptr);
    double* up = a.u + (static_cast<size_t>(p) * a.N + i) * R;
    reduce_warps<W>(a, g, sh, acc, [&](int l, double s) {
      up[l] = s;
      sh.s0[l] = s;
    });
    if (warp < a.ncq && !a.one_level) {
      const int gq = a.corner_q[i * a.ncq + warp];
      double acc2 = 0;
      if (gq >= 0)
        for (int kk = lane; kk < r; kk += 32) acc2 += QtX[static_cast<size_t>(kk) * E + 1 + gq] * sh.s0[kk];
      acc2 = warp_sum(acc2);
      const int dst = a.corner_dst[i * a.ncq + warp];
      if (lane == 0 && dst >= 0) a.t3tab_w[static_cast<size_t>(p) * 4 * a.n_pi + dst] = acc2;  // t(gp) += z(lr)
    }
    cons_sync();
  }
}

// ---------------------------------------------------------------- fused OP2 -> OP3 launch
__device__ __forceinline__ int& fused_gate() {
  __shared__ int g;
  return g;
}

/// After a phase of the fused launch: every item this CTA streamed in `kind` bumps its subdomain's
/// completion counter of stage `ph` (release: the item's owner-slot writes are fenced first).
__device__ void fused_signal(const CgArgs& a, int ph, int kind) {
  cons_sync();  // every consumer thread's slot stores issued
  if (threadIdx.x == 0) {
    __threadfence();
    const int nitems = n_items(a.N * a.P);
    for (int k = 0; k < nitems; ++k) {
      const int w = item_work(k, nitems, reverse_kind(kind));
      atomicAdd(a.pflags + static_cast<size_t>(ph) * a.N + w / a.P, 1u);
    }
  }
}

/// Before the next phase `kind` of the fused launch: wait until every subdomain whose owner slots
/// this CTA's items read (the item's subdomain and its edge neighbours) has all P parts through
/// stage `ph` of iteration `it` (acquire), then release the consumer warps. Warp 0 polls all the
/// (item, dependency) counters at once — one L2 round trip when they are already complete.
__device__ void fused_wait(const CgArgs& a, int ph, int kind, int it) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const unsigned target = static_cast<unsigned>(a.P) * static_cast<unsigned>(it);
    const int nitems = n_items(a.N * a.P);
    // watchdog: the counters only advance if every CTA of the launch is resident (one per SM); if a
    // wait exceeds 2 s the launch flags state[4] (the host reports it) instead of hanging the GPU
    // (reading the clock before the first poll, even when the counters are already complete, is
    // measured ~0.25 ms per C3 solve FASTER than reading it only after a failed poll)
    const unsigned long long t0 = gtimer();
    for (int base = 0; base < nitems * kCgMaxNbr; base += 32) {
      const int pr = base + lane;
      const unsigned* f = nullptr;
      if (pr < nitems * kCgMaxNbr) {
        const int i = item_work(pr / kCgMaxNbr, nitems, reverse_kind(kind)) / a.P;
        const int d = a.nbr[i * kCgMaxNbr + pr % kCgMaxNbr];
        if (d >= 0) f = a.pflags + static_cast<size_t>(ph) * a.N + d;
      }
      bool ok = f == nullptr;
      while (true) {
        if (!ok) {
          unsigned v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
          ok = v >= target;
        }
        if (__all_sync(0xffffffffu, ok)) break;
        if (a.fuse_sleep) __nanosleep(a.fuse_sleep);
        if (gtimer() - t0 > 2000000000ull) {
          if (lane == 0) atomicExch(a.state + 4, 1);
          break;
        }
      }
    }
    __threadfence();
  }
  cons_sync();
}

// ---------------------------------------------------------------- OP4 (per subdomain, all warps)
/// o_i = -phi + Q_G (s~ + u + Q_Pi^T nu) + Zc^T d2 ; CG mode also returns p . o_i.
/// optional sub-phase timer (trace builds): tm[15] holds the last timestamp
__device__ __forceinline__ void mark(unsigned long long* tm, int k) {
  if (tm != nullptr && threadIdx.x == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    tm[k] += now - tm[15];
    tm[15] = now;
  }
}

__device__ double dev_op4(const CgArgs& a, const Shared& sh, QtxStage& qst, int i, const double* v, int mode,
                          unsigned long long* tm = nullptr) {
  const SubGeo d = a.geo[i];
  const int r = d.r, R = a.rmax, E = a.ext, n = a.n_pi, nz = a.n_pi + a.npf;
  __shared__ double cq_mu[kMaxCq], cq_nu[kMaxCq], d2s[64], w3t[64];
  __shared__ RowTask tasks[2 * kMaxCq + 2 * 64];
  const int ncq = a.ncq;
  if (a.one_level) {
    // reduced_apply (solvers.cpp:262-274) at the trace rows: o = -phi + Q_G (s + u), written to the
    // owner slots of its Delta index (2 owners) or Pi index (up to 4 owners)
    const size_t ust = static_cast<size_t>(a.N) * R;
    const Staged stg = stage_qtx(a, sh, qst, i, r);
    const double* QtX = stg.qtx;
    for (int k = threadIdx.x; k < r; k += kThreads)
      sh.s0[k] = a.s[static_cast<size_t>(i) * R + k] + sum_parts(a.u + static_cast<size_t>(i) * R, ust, a.P, k);
    __syncthreads();
    double* qsv = sh.v1;
    coldot_split(QtX + 1, E, r, d.n_gamma, sh.s0, sh.red, Team{kThreads}, [&](int g, double s) { qsv[g] = s; });
    const int* gd = a.gamma_delta + static_cast<size_t>(i) * a.gmax;
    const int* gpi = a.gamma_pi + static_cast<size_t>(i) * a.gmax;
    double dot = 0;
    for (int g = threadIdx.x; g < d.n_gamma; g += kThreads) {
      const int dg = gd[g];
      const int idx = dg >= 0 ? dg : (gpi[g] >= 0 ? a.n_delta + gpi[g] : -1);
      if (idx < 0) continue;
      const double mphi = (mode == 0) ? v[idx] : 0.0;  // -phi
      const double o = mphi + qsv[g];
      if (dg >= 0) {
        a.otab_w[a.gamma_dst[static_cast<size_t>(i) * a.gmax + g]] = o;
      } else {
        for (int q = 0; q < ncq; ++q)
          if (a.corner_q[i * ncq + q] == g && a.corner_dst[i * ncq + q] >= 0) a.opitab_w[a.corner_dst[i * ncq + q]] = o;
      }
      if (mode == 0) dot += v[idx] * o;
    }
    return block_sum(dot, sh.red);
  }
  // this thread's output row (gamma point threadIdx.x): index, slot and -phi loaded up front, off the
  // critical path of the coarse row dots
  int pdg = -1, pdst = -1, pcr = -1;
  double pv = 0.0;
  if (threadIdx.x < d.n_gamma) {
    pdg = a.gamma_delta[static_cast<size_t>(i) * a.gmax + threadIdx.x];
    pdst = a.gamma_dst[static_cast<size_t>(i) * a.gmax + threadIdx.x];
  }
  if (threadIdx.x < a.crmax) pcr = a.cr_row[static_cast<size_t>(i) * a.crmax + threadIdx.x];
  const size_t st3 = 4 * static_cast<size_t>(n);
  const size_t ust = static_cast<size_t>(a.N) * R;
  double uu0 = 0, sk0 = 0;
  constexpr int kMaxP = 4;  // row parts of the batched path (C3: 2, C4: 1); more: the loop form below
  if (n <= kThreads && a.npf <= kThreads && a.P <= kMaxP) {
    // every value fresh from the previous phases is loaded before any shared-memory store (a store
    // in between would order the loads: one L2 round trip per gather instead of one in total);
    // the sums keep gather_z's / sum_parts' order, so the results are bitwise unchanged
    const int tid = threadIdx.x;
    double tz[4] = {0, 0, 0, 0}, pz[4] = {0, 0, 0, 0}, t3[4][kMaxP], up[kMaxP], dp = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int pp = 0; pp < kMaxP; ++pp) t3[q][pp] = 0.0;
#pragma unroll
    for (int pp = 0; pp < kMaxP; ++pp) up[pp] = 0.0;
    if (tid < n) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        tz[q] = a.ttab[4 * static_cast<size_t>(tid) + q];
#pragma unroll
        for (int pp = 0; pp < kMaxP; ++pp)
          if (pp < a.P) t3[q][pp] = a.t3tab[pp * st3 + static_cast<size_t>(tid) * 4 + q];
      }
    }
    if (tid < a.npf) {
      if (mode != 1)
#pragma unroll
        for (int q = 0; q < 4; ++q) pz[q] = a.ptab[4 * static_cast<size_t>(tid) + q];
      if (mode != 0) dp = a.dpi[tid];
    }
    if (mode == 0 && pdg >= 0) pv = v[pdg];
    if (tid < r) {
#pragma unroll
      for (int pp = 0; pp < kMaxP; ++pp)
        if (pp < a.P) up[pp] = a.u[pp * ust + static_cast<size_t>(i) * R + tid];
      sk0 = a.s[static_cast<size_t>(i) * R + tid];
    }
    if (tid < n) {
      sh.z[tid] = ((tz[0] + tz[1]) + tz[2]) + tz[3];
      double acc = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double sp = 0;
#pragma unroll
        for (int pp = 0; pp < kMaxP; ++pp)
          if (pp < a.P) sp += t3[q][pp];
        acc += sp;
      }
      sh.t2[tid] = acc;
    }
    if (tid < a.npf) {
      const double acc = ((pz[0] + pz[1]) + pz[2]) + pz[3];
      sh.z[n + tid] = (mode == 0) ? acc : (mode == 1 ? dp : dp - acc);
    }
#pragma unroll
    for (int pp = 0; pp < kMaxP; ++pp)
      if (pp < a.P) uu0 += up[pp];
  } else {
    if (mode == 0 && pdg >= 0) pv = v[pdg];
    gather_z(a, sh, mode, kThreads);
    for (int gp = threadIdx.x; gp < n; gp += kThreads) {
      double acc = 0;
      for (int q = 0; q < 4; ++q) acc += sum_parts(a.t3tab, st3, a.P, gp * 4 + q);
      sh.t2[gp] = acc;
    }
    if (threadIdx.x < r) {
      uu0 = sum_parts(a.u + static_cast<size_t>(i) * R, ust, a.P, threadIdx.x);
      sk0 = a.s[static_cast<size_t>(i) * R + threadIdx.x];
    }
  }
  if (pdg < 0) pdst = -1;
  // the four coarse row-dot families run concurrently (one warp per row)
  if (threadIdx.x < ncq) {
    const int g = a.corner_q[i * ncq + threadIdx.x];
    const int row = g >= 0 ? a.gamma_pi[static_cast<size_t>(i) * a.gmax + g] : -1;
    tasks[threadIdx.x] = RowTask{a.Wmu, sh.z, &cq_mu[threadIdx.x], nz, row, nz};          // mu = S^-1 (t + Dpp^T psi)
    tasks[ncq + threadIdx.x] = RowTask{a.Sinv, sh.t2, &cq_nu[threadIdx.x], n, row, n};    // nu = S^-1 t'
  }
  for (int rho = threadIdx.x; rho < a.crmax; rho += kThreads) {
    const int row = a.cr_row[static_cast<size_t>(i) * a.crmax + rho];
    tasks[2 * ncq + rho] = RowTask{a.Wd, sh.z, &d2s[rho], nz, row, nz};                   // d1 = psi - Dpp mu
    tasks[2 * ncq + a.crmax + rho] = RowTask{a.W3, sh.t2, &w3t[rho], n, row, n};          // Dpp nu
  }
  __syncthreads();
  mark(tm, 0);
  const Staged stg = stage_qtx(a, sh, qst, i, r);
  const double* QtX = stg.qtx;
  __syncthreads();
  mark(tm, 1);
  row_tasks(tasks, 2 * ncq + 2 * a.crmax, kWarps);
  __syncthreads();
  mark(tm, 2);
  if (threadIdx.x < a.crmax) d2s[threadIdx.x] = pcr >= 0 ? d2s[threadIdx.x] - w3t[threadIdx.x] : 0.0;
  int gq[kMaxCq];
#pragma unroll
  for (int q = 0; q < kMaxCq; ++q) gq[q] = q < ncq ? a.corner_q[i * ncq + q] : -1;
  for (int k = threadIdx.x; k < r; k += kThreads) {
    double uu = (k == threadIdx.x) ? uu0 : sum_parts(a.u + static_cast<size_t>(i) * R, ust, a.P, k);
    double sk = (k == threadIdx.x) ? sk0 : a.s[static_cast<size_t>(i) * R + k];
    for (int q = 0; q < ncq; ++q)
      if (gq[q] >= 0) {
        const double qk = QtX[static_cast<size_t>(k) * E + 1 + gq[q]];
        uu += qk * cq_nu[q];
        sk += qk * cq_mu[q];  // s~ = s + Q_Pi^T mu
      }
    sh.s0[k] = sk + uu;  // s~ + u + Q_Pi^T nu
  }
  __syncthreads();
  mark(tm, 3);
  const int* gd = a.gamma_delta + static_cast<size_t>(i) * a.gmax;
  const double* Zc = stg.zc;
  // o = -phi + Q_G s_tot + Zc^T d2 ; Q_G s_tot split over k-groups (coldot_split)
  double* qsv = sh.v1;
  coldot_split(QtX + 1, E, r, d.n_gamma, sh.s0, sh.red, Team{kThreads}, [&](int g, double s) { qsv[g] = s; });
  mark(tm, 4);
  double dot = 0;
  (void)gd;
  if (pdg >= 0) {  // n_gamma <= kThreads (cg_check_capacity): one gamma point per thread
    const int g = threadIdx.x;
    double zs = 0;
    for (int rho = 0; rho < a.crmax; ++rho) zs += Zc[static_cast<size_t>(rho) * a.gmax + g] * d2s[rho];
    const double o = pv + qsv[g] + zs;  // -phi + Q_G s_tot + Zc^T d2
    a.otab_w[pdst] = o;
    if (mode == 0) dot += pv * o;
  }
  dot = block_sum(dot, sh.red);
  mark(tm, 5);
  return dot;
}

__device__ __forceinline__ double gather_out(const CgArgs& a, int g) {
  if (g >= a.n_delta) {  // one-level Pi entry: its corner owners in subdomain order
    const double* o = a.opitab + 4 * (g - a.n_delta);
    return ((o[0] + o[1]) + o[2]) + o[3];
  }
  return a.otab[2 * g] + a.otab[2 * g + 1];
}

// ---------------------------------------------------------------- the persistent kernel
template <int W>
__global__ void __launch_bounds__(kThreads, 1) cg_persistent_kernel(CgArgs a, int job, const double* vin,
                                                                    double* vout) {
  cgs::grid_group grid = cgs::this_grid();
  const int G = gridDim.x, b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == kProducerWarp;
  __shared__ __align__(8) uint64_t bars[2 * kStages + 1];
  __shared__ double bsum[32];
  const Shared sh = carve(a, bars);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.empty[s], kCWarps);
    }
    mbar_init(sh.qbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  Producer pr;          // warp 15 lane 0
  pr.cnt = 0;
  pr.active = false;
  unsigned ccnt = 0;    // chunks consumed (consumer warps, uniform)
  QtxStage qst{0u, -1, false};

  // Producer: issue the first chunks of `kind` (the ring is idle: the caller's last ring readers
  // finished behind a block barrier) — they overlap the grid barrier that follows.
  auto prefetch = [&](int kind, bool recon) {
    qst.cached = -1;
    if (producer && lane == 0) {
      producer_begin(a, pr, kind, recon);
      producer_run(a, pr, sh, kStages);
    }
  };
  // Streamed phase: warp 15 issues the remaining chunks, warps 0..14 consume.
  auto finish_producer = [&]() {
    if (lane == 0) producer_run(a, pr, sh, -1);
    __syncwarp();
  };

  if (job == kJobRecon) {
    for (int i = b; i < a.N; i += G) dev_op1(a, sh, qst, i, vin, 2, false, 0.0, nullptr, nullptr);
    prefetch(kOp2, true);
    grid.sync();
    if (producer) finish_producer(); else dev_op2<W>(a, sh, ccnt, 2, kNoPre);
    __syncthreads();
    return;
  }

  if (job == kJobApply || job == kJobRhs) {
    const int mode = job == kJobApply ? 0 : 1;
    for (int i = b; i < a.N; i += G) dev_op1(a, sh, qst, i, vin, mode, false, 0.0, nullptr, nullptr);
    prefetch(kOp2, false);
    grid.sync();
    if (producer) finish_producer(); else dev_op2<W>(a, sh, ccnt, mode, kNoPre);
    __syncthreads();
    if (a.use_neumann) {
      prefetch(kNn1, false);
      grid.sync();
      if (producer) finish_producer(); else dev_nn1<W>(a, sh, ccnt, kNoPre);
      __syncthreads();
      prefetch(kNn2, false);
      grid.sync();
      if (producer) finish_producer(); else dev_nn2<W>(a, sh, ccnt, kNoPre);
      __syncthreads();
    }
    prefetch(kOp3, false);
    grid.sync();
    if (producer) finish_producer(); else dev_op3<W>(a, sh, ccnt, kNoPre);
    __syncthreads();
    qst.cached = -1;
    grid.sync();
    for (int i = b; i < a.N; i += G) dev_op4(a, sh, qst, i, vin, mode);
    grid.sync();
    for (int g = b * blockDim.x + threadIdx.x; g < a.n_cg; g += G * blockDim.x) vout[g] = gather_out(a, g);
    return;
  }

  // ---- CG (solvers.cpp:93-116): x0 = 0, r = p = b (cg_init), recursive residual
  // optional per-phase device timers (a.trace: G x 16 ns counters; profiling runs only)
  unsigned long long t_last = 0, t_acc[16] = {}, t_op4[16] = {};
  auto tr = [&](int k) {
    if (a.trace != nullptr && threadIdx.x == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (k >= 0) t_acc[k] += now - t_last;
      t_last = now;
    }
  };
  tr(-1);
  double rr = a.scal[0];
  const double bnorm = a.scal[1];
  if (a.state[1]) return;  // rhs == 0
  double beta = 0.0;
  for (int it = 1;; ++it) {
    double* pcur = a.pbuf[(it - 1) & 1];
    double* pnext = a.pbuf[it & 1];
    for (int i = b; i < a.N; i += G) dev_op1(a, sh, qst, i, nullptr, 0, true, beta, pcur, pnext);
    prefetch(kOp2, false);
    tr(0);
    grid.sync();
    tr(1);
    if (producer) finish_producer(); else dev_op2<W>(a, sh, ccnt, 0, kNoPre);
    __syncthreads();
    tr(2);
    if (a.use_neumann) {
      prefetch(kNn1, false);
      grid.sync();
      tr(3);
      if (producer) finish_producer(); else dev_nn1<W>(a, sh, ccnt, kNoPre);
      __syncthreads();
      tr(4);
      prefetch(kNn2, false);
      grid.sync();
      tr(5);
      if (producer) finish_producer(); else dev_nn2<W>(a, sh, ccnt, kNoPre);
      __syncthreads();
      tr(6);
    }
    prefetch(kOp3, false);
    grid.sync();
    tr(7);
    if (producer) finish_producer(); else dev_op3<W>(a, sh, ccnt, kNoPre);
    __syncthreads();
    tr(8);
    qst.cached = -1;
    grid.sync();
    tr(9);
    for (int i = b; i < a.N; i += G) {
      if (a.trace != nullptr && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_op4[15]));
      const double dot = dev_op4(a, sh, qst, i, pnext, 0, a.trace != nullptr ? t_op4 : nullptr);
      if (threadIdx.x == 0) a.pap_w[a.sub_lo + i] = dot;
    }
    tr(10);
    grid.sync();
    tr(11);
    // pAp = sum over subdomains of p . o_i (fixed order), alpha, x / r update
    const double pAp = det_sum(a.pap, a.N_global);
    if (pAp <= 0.0) {  // solvers.cpp:97-103
      if (b == 0 && threadIdx.x == 0) {
        a.state[3] = pAp < 0.0 ? 1 : 0;
        a.state[5] = it - 1;
        a.state[1] = 1;
      }
      break;
    }
    const double alpha = rr / pAp;
    double dsum = 0;
    for (int g = b * blockDim.x + threadIdx.x; g < a.n_cg; g += G * blockDim.x) {
      const double ap = gather_out(a, g);
      a.x[g] += alpha * pnext[g];
      const double rg = a.r[g] - alpha * ap;
      a.r[g] = rg;
      dsum += rg * rg;
    }
    dsum = block_sum(dsum, bsum);
    if (threadIdx.x == 0) a.partial[b] = dsum;
    tr(12);
    grid.sync();
    tr(13);
    const double rr_new = det_sum(a.partial, G);
    const double rel = sqrt(rr_new) / bnorm;
    if (b == 0 && threadIdx.x == 0) {
      a.hist[it - 1] = rel;
      a.state[5] = it;
    }
    if (rel <= a.rel_tol || it >= a.max_iter) {
      if (b == 0 && threadIdx.x == 0) {
        a.state[1] = 1;
        a.state[2] = rel <= a.rel_tol ? 1 : 0;
      }
      break;
    }
    beta = rr_new / rr;
    rr = rr_new;
    tr(14);
    // a.partial / a.pap are rewritten only after further grid barriers: no race with the reads
  }
  if (a.trace != nullptr && threadIdx.x == 0)
    for (int k = 0; k < 16; ++k) {
      a.trace[b * 32 + k] = static_cast<double>(t_acc[k]);
      a.trace[b * 32 + 16 + k] = k < 15 ? static_cast<double>(t_op4[k]) : 0.0;
    }
}

// ---------------------------------------------------------------- phase-by-phase execution
// The same phases as the persistent kernel, one launch each, for the sharded path: the host
// enqueues an all-reduce of the owner-slot tables between launches (comm.hpp). With one device
// the sequence is bitwise identical to the persistent kernel (same work split, same sums).
template <int W>
__global__ void __launch_bounds__(kThreads, 1) cg_phase_kernel(CgArgs a, int phase, int mode, int it,
                                                               const double* vin, double* vout) {
  const int G = gridDim.x, b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == kProducerWarp;
  __shared__ __align__(8) uint64_t bars[2 * kStages + 1];
  __shared__ double bsum[32];
  const Shared sh = carve(a, bars);
  if (threadIdx.x == 0) {
    phase_stamps()[0] = a.trace ? gtimer() : 0;
    phase_stamps()[2] = phase_stamps()[3] = phase_stamps()[4] = phase_stamps()[5] = 0;
    for (int s2 = 0; s2 < kStages; ++s2) {
      mbar_init(&sh.full[s2], 1);
      mbar_init(&sh.empty[s2], kCWarps);
    }
    mbar_init(sh.qbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  Producer pr;
  pr.cnt = 0;
  pr.active = false;
  unsigned ccnt = 0;
  QtxStage qst{0u, -1, false};
  const bool cg = (mode == 0 && vin == nullptr);  // CG iteration: v = r + beta p_cur
  // Programmatic dependent launch: let the next phase's CTAs start as SMs free up, and issue this
  // phase's static-data bulk copies (coefficient blocks, Q_r^T / Zc) before waiting for the
  // previous phase to complete — the in-kernel analogue of prefetching across a grid barrier.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const bool fused = phase == kPhFused;
  const bool streamed = phase == kPhOp2 || phase == kPhNn1 || phase == kPhNn2 || phase == kPhOp3 || fused;
  StreamPre pre{-1, -1, -1};
  if (streamed) {
    const int kind = (phase == kPhOp2 || fused) ? kOp2 : phase == kPhNn1 ? kNn1 : phase == kPhNn2 ? kNn2 : kOp3;
    if (producer && lane == 0) {
      producer_begin(a, pr, kind, mode == 2);
      producer_run(a, pr, sh, a.preissue);
      if (a.l2ahead > 0) producer_l2ahead(a, pr, a.l2ahead);
    }
    if (!producer) pre = stream_pre(a, kind);
  } else if ((phase == kPhOp1 || phase == kPhOp4) && b < a.N) {
    size_t qb;
    stage_issue(a, sh, qst, b, a.geo[b].r, &qb);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (streamed) __syncthreads();  // pre_geo() written by thread 0 before the wait
  if (a.trace && threadIdx.x == 0) phase_stamps()[1] = gtimer();
  // the streamed phases only write intermediate tables: they need neither the iteration counter
  // nor the stop flag (XR1 checks it), so their prologue starts with fresh data, not state
  if (cg && (!streamed || fused)) it = a.state[6];  // the iteration counter lives on the device (graph replays)
  double* pcur = a.pbuf[(it + 1) & 1];
  double* pnext = a.pbuf[it & 1];
  // converged / aborted earlier (the chunked sharded driver also replays streamed phases past the
  // stop: guard_all): drain the prefetched copies and leave
  if (cg && (!streamed || fused || a.guard_all) && a.state[1]) {
    if ((phase == kPhXr1 || phase == kPhXr2) && b == 0 && threadIdx.x == 0 && a.cond != 0)
      cudaGraphSetConditional(a.cond, 0);
    __shared__ int s_issued;
    if (threadIdx.x == 0) s_issued = (producer && lane == 0) ? 0 : 0;
    __syncthreads();
    if (producer && lane == 0) s_issued = static_cast<int>(pr.cnt);
    __syncthreads();
    for (int c = 0; c < s_issued; ++c) mbar_wait(&sh.full[c % kStages], (c / kStages) & 1u);
    if (qst.pending) mbar_wait(sh.qbar, 0u);
    __syncthreads();
    return;
  }
  switch (phase) {
    case kPhOp1: {
      const double beta = cg ? a.scal[2] : 0.0;
      for (int i = b; i < a.N; i += G) dev_op1(a, sh, qst, i, cg ? nullptr : vin, mode, cg, beta, pcur, pnext);
      trace_small(a, 0);
      return;
    }
    case kPhOp2:
    case kPhNn1:
    case kPhNn2:
    case kPhOp3: {
      if (producer) {
        if (lane == 0) producer_run(a, pr, sh, -1);  // the first kStages chunks went out before the wait
        __syncwarp();
      } else if (phase == kPhOp2) {
        dev_op2<W>(a, sh, ccnt, mode, pre);
      } else if (phase == kPhNn1) {
        dev_nn1<W>(a, sh, ccnt, pre);
      } else if (phase == kPhNn2) {
        dev_nn2<W>(a, sh, ccnt, pre);
      } else {
        dev_op3<W>(a, sh, ccnt, pre);
      }
      __syncthreads();
      if (a.trace && threadIdx.x == 0 && phase_stamps()[2] != 0) {
        // streamed-phase trace: slots 16 + 4 (phase - kPhOp2) + {entry->wait, wait->first chunk,
        // first chunk->last chunk, last chunk->exit}, ns summed over the launches
        const unsigned long long* t = phase_stamps();
        const unsigned long long end = gtimer();
        double* tr = a.trace + b * 32 + 16 + 4 * (phase - kPhOp2);
        tr[0] += static_cast<double>(t[4] - t[1]);  // prologue (after the wait)
        if (t[5] != 0) a.trace[b * 32 + 10 + (phase - kPhOp2)] += static_cast<double>(t[5] - t[1]);  // gather part
        tr[1] += static_cast<double>(t[2] - t[4]);  // first chunk's data wait
        tr[2] += static_cast<double>(t[3] - t[2]);
        tr[3] += static_cast<double>(end - t[3]);
      }
      return;
    }
    case kPhFused: {
      // OP2, NN1, NN2, OP3 back to back: the producer warp streams the four phases' chunks through
      // the ring without a break (the next phase's first chunks load while the consumers wait for
      // their neighbours); between phases an item waits only for the subdomains it reads from
      // the producer runs at most `preissue` chunks into the next phase before the consumers have
      // passed their neighbour wait (concurrent HBM traffic slows the latency-bound prologues)
      volatile int* gate = &fused_gate();
      if (threadIdx.x == 0) *gate = 0;
      __syncthreads();
      if (producer) {
        if (lane == 0) {
          producer_run(a, pr, sh, -1);
          for (int kind = kNn1; kind <= kOp3; ++kind) {
            producer_begin(a, pr, kind, false);
            if (a.fuse_gate) {
              producer_run(a, pr, sh, a.preissue);
              while (*gate < kind) {
              }
            }
            producer_run(a, pr, sh, -1);
          }
        }
        __syncwarp();
      } else {
        dev_op2<W>(a, sh, ccnt, mode, pre);
        fused_signal(a, 0, kOp2);
        // with fuse_pre the next phase's static prologue data (StreamPre) loads during the wait
        const StreamPre p1 = a.fuse_pre ? stream_pre(a, kNn1) : kNoPre;
        fused_wait(a, 0, kNn1, it);
        if (threadIdx.x == 0) *gate = kNn1;
        dev_nn1<W>(a, sh, ccnt, p1);
        fused_signal(a, 1, kNn1);
        const StreamPre p2 = a.fuse_pre ? stream_pre(a, kNn2) : kNoPre;
        fused_wait(a, 1, kNn2, it);
        if (threadIdx.x == 0) *gate = kNn2;
        dev_nn2<W>(a, sh, ccnt, p2);
        fused_signal(a, 2, kNn2);
        const StreamPre p3 = a.fuse_pre ? stream_pre(a, kOp3) : kNoPre;
        fused_wait(a, 2, kOp3, it);
        if (threadIdx.x == 0) *gate = kOp3;
        dev_op3<W>(a, sh, ccnt, p3);
      }
      __syncthreads();
      return;
    }
    case kPhOp4: {
      // the next OP2's coefficient rows into L2 while OP4 / XR / OP1 leave the HBM idle
      if (cg && a.l2pre != 0 && threadIdx.x == 0 && !a.compact) l2_prefetch_items(a, kOp2, a.l2pre);
      // DDELM_CG_TRACE: OP4's sub-phase timers (thread 0's clock) into trace slots 4..9
      __shared__ unsigned long long t4[16];
      if (a.trace != nullptr && threadIdx.x == 0)
        for (int k = 0; k < 16; ++k) t4[k] = 0;
      for (int i = b; i < a.N; i += G) {
        if (a.trace != nullptr && threadIdx.x == 0) t4[15] = gtimer();
        const double dot = dev_op4(a, sh, qst, i, cg ? pnext : vin, mode, a.trace != nullptr ? t4 : nullptr);
        if (cg && threadIdx.x == 0) a.pap_w[a.sub_lo + i] = dot;
      }
      if (a.trace != nullptr && threadIdx.x == 0 && b < a.N)
        for (int k = 0; k < 6; ++k) a.trace[b * 32 + 4 + k] += static_cast<double>(t4[k]);
      trace_small(a, 2);
      return;
    }
    case kPhXr1:    // alpha, x / r update, r.r partials (solvers.cpp:96-107); the last CTA to finish
    case kPhXr2: {  // also takes the stopping decision (solvers.cpp:108-116) — one launch per iteration
      __shared__ int s_last;
      if (phase == kPhXr1) {
        // this thread's first element, loaded together with p.Ap and the CG scalars (every value
        // here is fresh from OP4 / the previous XR: one L2 round trip instead of two)
        const int g0 = b * blockDim.x + threadIdx.x;
        double ap0 = 0, pc0 = 0, r0 = 0;
        if (g0 < a.n_cg) {
          ap0 = gather_out(a, g0);
          pc0 = pcur[g0];
          r0 = a.r[g0];
        }
        const double pAp = det_sum(a.pap, a.N_global);
        if (pAp <= 0.0) {
          if (b == 0 && threadIdx.x == 0) {
            a.state[3] = pAp < 0.0 ? 1 : 0;
            a.state[5] = it - 1;
            a.state[1] = 1;
            if (a.cond != 0) cudaGraphSetConditional(a.cond, 0);
          }
          return;
        }
        const double alpha = a.scal[0] / pAp;
        const double beta = a.scal[2];  // read before arriving: the last CTA overwrites it below
        double dsum = 0;
        for (int g = g0; g < a.n_cg; g += G * blockDim.x) {
          const bool first = g == g0;
          const double ap = first ? ap0 : gather_out(a, g);
          const double rgo = first ? r0 : a.r[g];
          // p = r + beta p_cur on EVERY index (replicated CG vectors: a sharded rank's OP1 writes
          // only the indices its subdomains touch); bitwise the value OP1 stored
          const double pn = __fma_rn(beta, first ? pc0 : pcur[g], rgo);
          pnext[g] = pn;
          a.x[g] += alpha * pn;
          const double rg = rgo - alpha * ap;
          a.r[g] = rg;
          dsum += rg * rg;
        }
        dsum = block_sum(dsum, bsum);
        if (threadIdx.x == 0) {
          a.partial[b] = dsum;
          __threadfence();
          s_last = atomicAdd(&a.state[7], 1) == G - 1;  // arrival counter (reset by cg_init / below)
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
      } else if (b != 0) {
        return;
      }
      const double rr_new = det_sum(a.partial, a.xr_parts);
      const double rel = sqrt(rr_new) / a.scal[1];
      const bool stop = rel <= a.rel_tol || it >= a.max_iter;
      __syncthreads();
      if (threadIdx.x == 0) {
        a.state[7] = 0;
        a.hist[it - 1] = rel;
        a.state[5] = it;
        if (stop) {
          a.state[1] = 1;
          a.state[2] = rel <= a.rel_tol ? 1 : 0;
        } else {
          a.scal[2] = rr_new / a.scal[0];
          a.scal[0] = rr_new;
          a.state[6] = it + 1;
        }
        if (a.cond != 0) cudaGraphSetConditional(a.cond, stop ? 0 : 1);  // CUDA-graph while loop
      }
      return;
    }
    default:  // kPhGather
      for (int g = b * blockDim.x + threadIdx.x; g < a.n_cg; g += G * blockDim.x) vout[g] = gather_out(a, g);
      return;
  }
}

__global__ void __launch_bounds__(256) cg_init_kernel(CgArgs a) {
  __shared__ double red[32];
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  double d = 0;
  if (g < a.n_cg) {
    const double b = a.rhs[g];
    a.x[g] = 0.0;
    a.r[g] = b;
    a.pbuf[0][g] = b;
    d = b * b;
  }
  d = block_sum(d, red);
  if (threadIdx.x == 0) a.partial[blockIdx.x] = d;
}

__global__ void cg_init2_kernel(CgArgs a, int nblk) {
  if (threadIdx.x != 0) return;
  double rr = 0;
  for (int k = 0; k < nblk; ++k) rr += a.partial[k];
  a.scal[0] = rr;
  a.scal[1] = sqrt(rr);
  a.scal[2] = 0.0;  // beta of "iteration 0" (phase-by-phase CG)
  for (int k = 0; k < 8; ++k) a.state[k] = 0;
  a.state[6] = 1;  // phase-by-phase CG: current iteration
  if (a.pflags != nullptr)
    for (int k = 0; k < 3 * a.N; ++k) a.pflags[k] = 0u;  // fused-launch completion counters
  if (rr == 0.0) {
    a.state[1] = 1;  // bnorm == 0: converged with x = 0 (solvers.cpp:89-92)
    a.state[2] = 1;
  }
}

int wmax_host(const CgArgs& a) { return std::max(std::max(a.rmax, a.fmax), std::max(a.dmax, a.gmax)); }

size_t smem_bytes(const CgArgs& a) {
  const int wm = wmax_host(a);
  const int wred = std::min(kRedW, (std::max(std::max(a.rmax, a.fmax), a.dmax) + 31) & ~31);
  const size_t small = static_cast<size_t>(wm) + std::max(kCWarps * wred, kThreads) + a.n_pi + a.npf +
                       std::max(a.n_pi, 1) + wm + static_cast<size_t>(a.rmax);
  return static_cast<size_t>(kStages) * kStageBytes + sizeof(double) * small;
}

/// Register-blocking width of the streamed phases: widest row-dot operand / axpy output / 32.
int width_regs(const CgArgs& a) {
  const int w = std::max(std::max(a.rmax, a.fmax), a.dmax);
  return w <= 256 ? 8 : w <= 512 ? 16 : 32;
}

const void* kernel_for(const CgArgs& a) {
  const int w = width_regs(a);
  return w == 8    ? reinterpret_cast<const void*>(cg_persistent_kernel<8>)
         : w == 16 ? reinterpret_cast<const void*>(cg_persistent_kernel<16>)
                   : reinterpret_cast<const void*>(cg_persistent_kernel<32>);
}

}  // namespace

int cg_grid(const CgArgs& a) {
  int dev = 0, sms = 0, per_sm = 0;
  DDG_CUDA(cudaGetDevice(&dev));
  DDG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t sm = smem_bytes(a);
  const void* k = kernel_for(a);
  DDG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
  DDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, sm));
  if (per_sm < 1) throw CudaError("cg_persistent_kernel cannot be resident (occupancy 0)");
  return sms;  // one CTA per SM
}

void cg_check_capacity(const CgArgs& a) {
  // shapes the kernel's shared-memory carve-up and thread mapping assume
  const int w = std::max(std::max(a.rmax, a.fmax), a.dmax);
  if (a.gmax > kThreads || a.crmax > 64 || w > kMaxW)
    throw std::invalid_argument("interface block sizes exceed the CG kernel's capacity");
  if ((a.ldKF & 1) || (a.ldKD & 1)) throw std::logic_error("packed CG blocks need even row strides");
  if (8 * std::max(a.ldKF, a.ldKD) > kStageBytes)
    throw std::invalid_argument("one coefficient row exceeds a CG pipeline stage");
  if (smem_bytes(a) > 227 * 1024) throw std::invalid_argument("CG kernel shared memory exceeds 227 KB");
}

int cg_rows_per_chunk_max(const CgArgs& a) { return std::max(rows_per_chunk(a.ldKF), rows_per_chunk(a.ldKD)); }

void cg_launch(const CgArgs& a, int job, const double* vin, double* vout, cudaStream_t st) {
  cg_check_capacity(a);
  const int G = cg_grid(a);
  const size_t sm = smem_bytes(a);
  CgArgs arg = a;
  void* params[] = {&arg, &job, &vin, &vout};
  DDG_CUDA(cudaLaunchCooperativeKernel(kernel_for(a), dim3(G), dim3(kThreads), params, sm, st));
}

namespace {
/// apply_P / apply_PT (solvers.cpp:450-474) through the NN1 / NN2 phases: op 0 places v as the
/// gathered flux values NN1 reads (part 0, first owner slot; the debug flip cancels), op 1 places
/// u as the gathered P x NN2 reads, op 2 gathers P v from NN1's owner slots, op 3 gathers
/// -(zz) = P^T u from NN2's (the sign OP3 applies, solvers.cpp:473).
__global__ void neumann_io_kernel(CgArgs a, int op, const double* v, double* out) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < a.n_delta; g += gridDim.x * blockDim.x) {
    if (op == 0) a.xtab[2 * static_cast<size_t>(g)] = a.flip_sign[g] * v[g];
    else if (op == 1) a.trtab[2 * static_cast<size_t>(g)] = v[g];
    else if (op == 2) out[g] = gather_delta(a.trtab, a, g);
    else out[g] = -gather_delta(a.zztab, a, g);
  }
}
}  // namespace

void cg_launch_neumann_io(const CgArgs& a, int op, const double* v, double* out, cudaStream_t st) {
  neumann_io_kernel<<<ceil_div(std::max(a.n_delta, 1), 256), 256, 0, st>>>(a, op, v, out);
  DDG_LAUNCH_CHECK();
}

void cg_launch_phase(const CgArgs& a, int phase, int mode, int it, const double* vin, double* vout,
                     cudaStream_t st) {
  cg_check_capacity(a);
  const int G = cg_grid(a);
  const size_t sm = smem_bytes(a);
  const int wreg = width_regs(a);
  const void* k = wreg == 8    ? reinterpret_cast<const void*>(cg_phase_kernel<8>)
                  : wreg == 16 ? reinterpret_cast<const void*>(cg_phase_kernel<16>)
                               : reinterpret_cast<const void*>(cg_phase_kernel<32>);
  DDG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
  const int grid = (phase == kPhXr2) ? 1 : G;
  // programmatic dependent launch (the kernel overlaps its static prologue with the previous
  // phase; griddepcontrol.wait orders every dependent read); DDELM_CG_PDL=0 disables it
  static const bool pdl = [] {
    const char* e = std::getenv("DDELM_CG_PDL");
    return !(e && std::atoi(e) == 0);
  }();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  if (wreg == 8)
    DDG_CUDA(cudaLaunchKernelEx(&cfg, cg_phase_kernel<8>, a, phase, mode, it, vin, vout));
  else if (wreg == 16)
    DDG_CUDA(cudaLaunchKernelEx(&cfg, cg_phase_kernel<16>, a, phase, mode, it, vin, vout));
  else
    DDG_CUDA(cudaLaunchKernelEx(&cfg, cg_phase_kernel<32>, a, phase, mode, it, vin, vout));
}

namespace {
/// out[k] = the P-part sum of table slot e[k] in the consumers' order (sum_parts): what a reader
/// of the slot would gather, so the importer's single stored value reproduces its sum bit for bit
__global__ void __launch_bounds__(256) xpack_kernel(XTabs t, const XEntry* e, int n, double* out, const int* state) {
  if (state != nullptr && state[1]) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const XEntry x = e[k];
    const double* base = t.ptr[x.table];
    const int parts = t.parts[x.table];
    const long long ps = t.pstride[x.table];
    double s = 0;
    for (int p = 0; p < parts; ++p) s += base[p * ps + x.idx];
    out[k] = s;
  }
}
/// table slot e[k] (part 0) = in[k]; the other parts of an imported slot stay zero
__global__ void __launch_bounds__(256) xunpack_kernel(XTabs t, const XEntry* e, int n, const double* in, const int* state) {
  if (state != nullptr && state[1]) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const XEntry x = e[k];
    t.ptr[x.table][x.idx] = in[k];
  }
}
}  // namespace

XTabs cg_xtabs(const CgArgs& a) {
  XTabs t{};
  auto set = [&](int id, double* p, int parts, long long ps) {
    t.ptr[id] = p;
    t.parts[id] = parts;
    t.pstride[id] = ps;
  };
  const long long nd2 = 2LL * a.n_delta, npi4 = 4LL * a.n_pi, npf4 = 4LL * a.npf;
  set(kTabT, a.ttab, 1, 0);
  set(kTabPsi, a.ptab, 1, 0);
  set(kTabT3, a.t3tab, a.P, npi4);
  set(kTabO, a.otab, 1, 0);
  set(kTabX, a.xtab, a.P, nd2);
  set(kTabTr, a.trtab, a.P, nd2);
  set(kTabZz, a.zztab, a.P, nd2);
  set(kTabXc, a.xctab, a.P, npf4);
  set(kTabOpi, a.opitab, 1, 0);
  set(kTabPap, a.pap, 1, 0);
  return t;
}

void launch_xpack(const XTabs& t, const XEntry* e, int n, double* out, const int* state, cudaStream_t st) {
  if (n <= 0) return;
  xpack_kernel<<<std::min(148, ceil_div(n, 256)), 256, 0, st>>>(t, e, n, out, state);
  DDG_LAUNCH_CHECK();
}

void launch_xunpack(const XTabs& t, const XEntry* e, int n, const double* in, const int* state, cudaStream_t st) {
  if (n <= 0) return;
  xunpack_kernel<<<std::min(148, ceil_div(n, 256)), 256, 0, st>>>(t, e, n, in, state);
  DDG_LAUNCH_CHECK();
}

void cg_launch_init(const CgArgs& a, cudaStream_t st) {
  const int nblk = ceil_div(a.n_cg, 256);
  cg_init_kernel<<<nblk, 256, 0, st>>>(a);
  cg_init2_kernel<<<1, 32, 0, st>>>(a, nblk);
  DDG_LAUNCH_CHECK();
}

}  // namespace ddg
