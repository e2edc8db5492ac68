// FSA-based fast beam search (Algorithm 1 of arXiv 2211.00484), persistent
// and stream-stationary like decode.cu.  Restates fsa_search.hpp:
//
//   get_contexts  (124-154)  distinct contexts of a stream's active tuples,
//                            ascending (active is kept sorted by (ctx, state))
//   joiner + log-softmax     exact fp32 logits (decode_common.cuh) and the
//                            row normaliser; lp[k] = double(l_k) - lse as in
//                            model.hpp:115-125
//   expand_arcs   (161-223)  blank self-candidate and one candidate per
//                            outgoing graph arc, read from 16-byte CSR arc
//                            records; duplicates (ctx, state) merged by MAX
//   prune_streams (230-297)  (score desc, ctx asc, state asc) order,
//                            inclusive beam floor, max_states, then the first
//                            max_contexts contexts; survivors numbered in
//                            (ctx, state) order; every raw arc into a survivor
//                            is kept, in generation order
//   best_path     (fsa.hpp:345-376) on the HBM lattice after the last frame:
//                            backward tropical suffix maxima, forward trace
//                            taking the first arc that attains the remainder.
//
// Candidate selection without materialising all candidates: the top
// max_states distinct keys all score >= the M-th largest raw candidate once
// the raw candidates at or above that threshold hold >= max_states distinct
// keys.  A per-stream 256-bin score histogram below the stream's best finds
// such a threshold; only candidates above it enter a shared-memory hash
// (key -> max score, atomicMax on order-preserving integers), whose distinct
// entries are bitonic-sorted.  This is exact, not approximate: every key with
// max >= threshold is present with its true max.
#include <algorithm>

#include "decode_common.cuh"

namespace rnntg {
namespace {

using namespace dec;

constexpr int kMaxStates = kFsaMaxStates;  // device cap on max_states
constexpr int kHashCap = 256;    // hot-candidate hash entries per stream
constexpr int kBins = 256;
constexpr int kSurvHash = 128;
constexpr int kMaxRaw = 32768;   // raw candidates per stream-frame (64 states x 511 arcs)
constexpr uint64_t kEmptyKey = ~0ull;

struct ArcRec {  // matches the host ArcRec in capi.cu
  int32_t dst, label;
  double w;
};

struct LatArc {  // one lattice arc
  int32_t src, dst, label, pad;
  double score;
};

struct FsaStream {
  unsigned long long raw_total, lat_total;  // counters (group thread 0)
  int32_t n_act, num_nodes, nrows, row_base;
  int32_t n_raw, n_hot, n_sort, n_surv;
  int32_t bstar, arc_count, arc_off, flag;
  unsigned long long m_first, m_keep;  // prune: first-occurrence / survivor masks over sorted entries
  double best, floor;
  int32_t act_ctx[kMaxStates], act_state[kMaxStates], act_node[kMaxStates], act_row[kMaxStates];
  double act_score[kMaxStates];
  int32_t act_off[kMaxStates + 1];
  int32_t act_abase[kMaxStates];  // first CSR arc of the tuple's graph state
  int32_t act_shift[kMaxStates];  // (ctx % V) * V: the tuple's context shifted for a token (a1)
  double ub;                      // upper bound on the frame's best candidate
  uint32_t mbits[kMaxRaw / 32];   // raw candidates that enter the lattice
  int32_t row_ctx[kMaxStates];
  int32_t bins[kBins];
  uint64_t hkey[kHashCap];
  unsigned long long hval[kHashCap];
  uint64_t s1[kHashCap], s2[kHashCap];  // compacted hot entries (~score, key)
  int32_t surv_ctx[kMaxStates], surv_state[kMaxStates];
  double surv_score[kMaxStates];
  uint64_t shkey[kSurvHash];
  int32_t shnode[kSurvHash];
  double red_d[16];
  int32_t red_i[16];
#if RNNTG_FSA_PASS_CLOCKS
  long long pclk[8], pclk_last;
#endif
};

struct FsaSmem {
  uint64_t etab[256];            // glibc exp table (lse_exact)
  WPipe pipe;                    // in smem: no registers pinned across the frame loop
  unsigned long long rows_total;
  long long ph[3];               // thread 0: h build, joiner GEMM, lse + expand/prune
  uint64_t bar[2];
  uint32_t wcur[2];
  int64_t row_pe[kRowCap];
  int32_t row_ctx[kRowCap];
  double row_lse[kRowCap];
  double row_lpmax[kRowCap];  // max_k lp[k] of the row
  float row_m[kRowCap];       // row maxima (lse_rows_cta)
  int32_t nrows;
};

__device__ __forceinline__ unsigned long long ord_of(double x) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dbl_of(unsigned long long o) {
  const unsigned long long u = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  return __longlong_as_double(static_cast<long long>(u));
}
__device__ __forceinline__ uint64_t key_of(int32_t ctx, int32_t state) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(ctx)) << 32) | static_cast<uint32_t>(state);
}
__device__ __forceinline__ uint32_t hash_slot(uint64_t k, uint32_t cap) {
  k ^= k >> 29;
  k *= 0xbf58476d1ce4e5b9ull;
  k ^= k >> 32;
  return static_cast<uint32_t>(k) & (cap - 1);
}

// Thread-group helpers (G groups of NT = 512/G threads; named barrier 1+grp).
struct Group {
  int id, tid, nt;
  __device__ __forceinline__ void sync() const {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + id), "r"(nt) : "memory");
  }
};

__device__ double group_max(const Group& g, FsaStream& S, double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = g.tid >> 5, nw = g.nt >> 5;
  if ((g.tid & 31) == 0) S.red_d[w] = v;
  g.sync();
  double r = S.red_d[0];
  for (int i = 1; i < nw; ++i) r = fmax(r, S.red_d[i]);
  g.sync();
  return r;
}

// Exclusive scan of one int per thread over the group; returns the prefix,
// *total gets the sum.
__device__ int group_scan(const Group& g, FsaStream& S, int v, int* total) {
  const int lane = g.tid & 31, w = g.tid >> 5, nw = g.nt >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  if (lane == 31) S.red_i[w] = incl;
  g.sync();
  int base = 0, tot = 0;
  for (int i = 0; i < nw; ++i) {
    if (i < w) base += S.red_i[i];
    tot += S.red_i[i];
  }
  g.sync();
  *total = tot;
  return base + incl - v;
}

// Raw candidate q of the stream (generation order of expand_arcs): active
// tuple i = the segment of q; q == act_off[i] is its blank self-candidate,
// otherwise graph arc (q - act_off[i] - 1) of its state.
struct Raw {
  int32_t i, ctx, state, label;
  double arc_score, score;
};

// Where a candidate's log-probability comes from: the joiner's logits in
// shared memory and the row's exact normaliser (the decoder), or the
// caller's log-prob rows (the step API, expand_arcs' plug-in point,
// fsa_search.hpp:59-61).  lp(row, label) = double(l) - lse, as
// log_softmax_row writes it (model.hpp:115-125).
struct LpJoiner {
  const float* L;
  const double* lse;
  int Vp;
  __device__ __forceinline__ double lp(int row, int label) const {
    return static_cast<double>(L[static_cast<int64_t>(row) * Vp + label]) - lse[row];
  }
};
struct LpRows {
  const double* P;
  int V;
  __device__ __forceinline__ double lp(int row, int label) const { return P[static_cast<int64_t>(row) * V + label]; }
};

// The active tuple whose candidate segment holds q: the last i < n_act with
// act_off[i] <= q (act_off[0] = 0, strictly increasing), by binary lifting
// over kMaxStates -- a fixed, unrolled sequence of predicated loads, so a
// thread's kU lookups interleave instead of running data-dependent loops.
__device__ __forceinline__ int seg_of(const FsaStream& S, int q) {
  int lo = 0;
#pragma unroll
  for (int step = kMaxStates / 2; step > 0; step >>= 1) {
    const int mid = lo + step;
    if (mid < S.n_act && S.act_off[mid] <= q) lo = mid;
  }
  return lo;
}

template <class Src>
__device__ __forceinline__ Raw raw_cand(const FsaStream& S, int q, const ArcRec* __restrict__ arcs, const Src& src,
                                        int V) {
  const int lo = seg_of(S, q);
  Raw r;
  r.i = lo;
  const int row = S.row_base + S.act_row[lo];
  const double sc = S.act_score[lo];
  const int j = q - S.act_off[lo];
  if (j == 0) {
    r.ctx = S.act_ctx[lo];
    r.state = S.act_state[lo];
    r.label = 0;
    r.arc_score = src.lp(row, 0);
  } else {
    const ArcRec a = arcs[S.act_abase[lo] + j - 1];
    r.ctx = S.act_shift[lo] + a.label;
    r.state = a.dst;
    r.label = a.label;
    r.arc_score = a.w + src.lp(row, a.label);
  }
  r.score = sc + r.arc_score;
  return r;
}

// kU raw candidates q0, q0+stride, ... at once: all locations first, then
// all (independent) 16-byte arc loads, then the arithmetic, so a thread has
// kU L2 requests in flight instead of one.
constexpr int kU = 4;
template <class Src>
__device__ __forceinline__ void raw_batch(const FsaStream& S, int q0, int stride, int nraw,
                                          const ArcRec* __restrict__ arcs, const Src& src, int V, Raw (&r)[kU],
                                          bool (&ok)[kU]) {
  int ii[kU], jj[kU];
  ArcRec a[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int q = q0 + u * stride;
    ok[u] = q < nraw;
    const int lo = seg_of(S, q);
    ii[u] = lo;
    jj[u] = ok[u] ? q - S.act_off[lo] : 0;
  }
#pragma unroll
  for (int u = 0; u < kU; ++u)
    if (jj[u] > 0) a[u] = arcs[S.act_abase[ii[u]] + jj[u] - 1];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const int lo = ii[u];
    const int row = S.row_base + S.act_row[lo];
    r[u].i = lo;
    if (jj[u] == 0) {
      r[u].ctx = S.act_ctx[lo];
      r[u].state = S.act_state[lo];
      r[u].label = 0;
      r[u].arc_score = src.lp(row, 0);
    } else {
      r[u].ctx = S.act_shift[lo] + a[u].label;
      r[u].state = a[u].dst;
      r[u].label = a[u].label;
      r[u].arc_score = a[u].w + src.lp(row, a[u].label);
    }
    r[u].score = S.act_score[lo] + r[u].arc_score;
  }
}

// Histogram bin of a candidate below the stream's upper bound `ub`
// (monotone non-increasing in the score); kBins = beyond the binned range.
__device__ __forceinline__ int ub_bin(double ub, double score, double scale) {
  const double d = (ub - score) * scale;
  return d < 0.0 ? 0 : (d < kBins ? static_cast<int>(d) : kBins);
}

// One frame of expand_arcs + prune_streams (fsa_search.hpp:161-297) for the
// stream of thread group `grp`, its active tuples in S (their joiner rows
// S.row_base + act_row), log-probs from `src`, row_lpmax[r] = max_k lp(r, k):
// the new active set in S, the frame's lattice arcs in the pool, its frame
// info in *finfo_t, the new nodes' contexts in nctx.  Shared by the decoder
// (fsa_kernel, LpJoiner) and the step API (fsa_step_kernel, LpRows).
// Development: RNNTG_FSA_PASS_CLOCKS=1 accumulates group 0's per-pass cycles
// into fsa_pass_clk (read by tools/prof_fsa.py through rnntg_get_stats? no:
// through the counters slots 12..15 and 5-7 at kernel end).
#ifndef RNNTG_FSA_PASS_CLOCKS
#define RNNTG_FSA_PASS_CLOCKS 0
#endif
#if RNNTG_FSA_PASS_CLOCKS
#define FSA_MARK(i)                                   \
  do {                                                \
    if (grp.tid == 0 && grp.id == 0) {                \
      const long long now_ = clock64();               \
      S.pclk[i] += now_ - S.pclk_last;                \
      S.pclk_last = now_;                             \
    }                                                 \
  } while (0)
#else
#define FSA_MARK(i) \
  do {              \
  } while (0)
#endif

template <class Src>
__device__ __forceinline__ void fsa_frame(FsaStream& S, const Group& grp, const Src& src,
                                          const double* __restrict__ row_lpmax, int V,
                                          const ArcRec* __restrict__ arcs, const int32_t* __restrict__ gsplits,
                                          const double* __restrict__ gmaxw, double beam, int K, int max_states,
                                          int max_contexts, int M, double scale, LatArc* __restrict__ lat,
                                          int64_t lat_cap, unsigned long long* __restrict__ lat_count,
                                          int4* __restrict__ finfo_t, int32_t* __restrict__ nctx,
                                          int32_t* __restrict__ error_flag) {
  const int nt = grp.nt;
      // ---- expand_arcs ----
      // Segment offsets of the raw candidates (one thread per active tuple,
      // group scan) and an upper bound on the frame's best candidate: tuple i
      // scores at most score_i + max(0, max arc weight of its state) +
      // max_k lp_i[k].
      int n_raw_all = 0;  // every thread's copy of the group scan total
      {
        const int i = grp.tid;
        int cnt = 0;
        double bound = -INFINITY;
        if (i < S.n_act) {
          const int st = S.act_state[i];
          const int a0 = gsplits[st], a1 = gsplits[st + 1];
          S.act_abase[i] = a0;
          S.act_shift[i] = (S.act_ctx[i] % V) * V;
          cnt = 1 + a1 - a0;
          bound = S.act_score[i] + fmax(0.0, gmaxw[st]) + row_lpmax[S.row_base + S.act_row[i]];
        }
        int total = 0;
        const int off = group_scan(grp, S, cnt, &total);
        n_raw_all = total;
        if (i < S.n_act) S.act_off[i] = off;
        const double ubm = group_max(grp, S, bound);
        if (grp.tid == 0) {
          S.act_off[S.n_act] = total;
          S.n_raw = total;
          S.ub = ubm + 1e-9 * fabs(ubm) + 1e-12;  // absorbs the rounding of the bound itself
          if (total > kMaxRaw) atomicExch(error_flag, 6);
        }
      }
      for (int b = grp.tid; b < kBins; b += nt) S.bins[b] = 0;
      for (int b = grp.tid; b < kHashCap; b += nt) {
        S.hkey[b] = kEmptyKey;
        S.hval[b] = 0ull;
      }
      // (the scan total, not S.n_raw: thread 0 may still be writing that)
      for (int w = grp.tid; w < (min(n_raw_all, kMaxRaw) + 31) / 32; w += nt) S.mbits[w] = 0u;
      grp.sync();
      const int nraw = min(S.n_raw, kMaxRaw);
      const double ub = S.ub;
      if (grp.tid == 0) S.raw_total += nraw;
      FSA_MARK(0);  // segment offsets, bound, clears
      // Pass A: the stream's best candidate and a histogram below `ub`.
      double mx = -INFINITY;
      for (int q0 = grp.tid; q0 < nraw; q0 += kU * nt) {
        Raw rc[kU];
        bool ok[kU];
        raw_batch(S, q0, nt, nraw, arcs, src, V, rc, ok);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (!ok[u]) continue;
          mx = fmax(mx, rc[u].score);
          const int b = ub_bin(ub, rc[u].score, scale);
          if (b < kBins) atomicAdd(&S.bins[b], 1);
        }
      }
      const double best = group_max(grp, S, mx);
      const double floor = best - beam;  // prune_streams 247-248
      // Smallest prefix of bins lying wholly at or above the floor that holds
      // M candidates; kBins = every candidate at or above the floor.  The bins
      // become inclusive prefix counts (a group scan over contiguous runs of
      // bins); bin b qualifies if it lies above the floor and its prefix
      // reaches M, and validity is monotone in b, so bstar = the smallest
      // qualifying bin.
      {
        constexpr int kMaxRun = kBins / 128;  // nt >= 128
        const int run = kBins / nt > 0 ? kBins / nt : 1;
        const int b0 = grp.tid * run;
        int loc[kMaxRun > 0 ? kMaxRun : 1];
        int sum = 0;
#pragma unroll
        for (int j = 0; j < (kMaxRun > 0 ? kMaxRun : 1); ++j) {
          loc[j] = (j < run && b0 + j < kBins) ? S.bins[b0 + j] : 0;
          sum += loc[j];
        }
        if (grp.tid == 0) {
          S.bstar = kBins;
          S.n_hot = 0;
        }
        int total = 0;
        int cum = group_scan(grp, S, sum, &total);
#pragma unroll
        for (int j = 0; j < (kMaxRun > 0 ? kMaxRun : 1); ++j) {
          const int b = b0 + j;
          if (j < run && b < kBins) {
            cum += loc[j];
            S.bins[b] = cum;
            if (cum >= M && !(ub - (b + 1) / scale < floor)) atomicMin(&S.bstar, b);
          }
        }
      }
      grp.sync();
      FSA_MARK(1);  // pass A + threshold
      // Pass B: hot candidates into the hash; widen the threshold if
      // duplicates left fewer than K distinct keys.
      while (true) {
        const int bstar = S.bstar;
        for (int q0 = grp.tid; q0 < nraw; q0 += kU * nt) {
          Raw rc[kU];
          bool ok[kU];
          raw_batch(S, q0, nt, nraw, arcs, src, V, rc, ok);
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            if (!ok[u] || rc[u].score < floor) continue;
            if (bstar < kBins && ub_bin(ub, rc[u].score, scale) > bstar) continue;
            const uint64_t k = key_of(rc[u].ctx, rc[u].state);
            uint32_t slot = hash_slot(k, kHashCap);
            for (int probe = 0; probe < kHashCap; ++probe) {
              const uint64_t prev = atomicCAS(reinterpret_cast<unsigned long long*>(&S.hkey[slot]),
                                              static_cast<unsigned long long>(kEmptyKey),
                                              static_cast<unsigned long long>(k));
              if (prev == kEmptyKey) atomicAdd(&S.n_hot, 1);
              if (prev == kEmptyKey || prev == k) {
                atomicMax(&S.hval[slot], ord_of(rc[u].score));
                break;
              }
              slot = (slot + 1) & (kHashCap - 1);
              if (probe == kHashCap - 1) atomicExch(error_flag, 3);
            }
          }
        }
        grp.sync();
        if (S.n_hot >= K || bstar >= kBins) break;
        if (S.n_hot > kHashCap / 2) break;
        grp.sync();
        if (grp.tid == 0) {  // widen by another M candidates (max is idempotent)
          int b = bstar + 1;
          for (; b < kBins; ++b) {
            if (ub - (b + 1) / scale < floor) {
              b = kBins;
              break;
            }
            if (S.bins[b] - S.bins[bstar] >= M) break;  // bins hold prefix counts
          }
          S.bstar = min(b, kBins);
        }
        grp.sync();
      }
      if (grp.tid == 0 && S.n_hot > kHashCap * 3 / 4) atomicExch(error_flag, 3);
      FSA_MARK(2);  // pass B
      // Compact the distinct keys; the first min(K, D) of them in (score
      // desc, key asc) order are found by rank (each entry counts the
      // entries before it: keys are distinct, so ranks are too) and land in
      // hkey / hval[rank] (the hash is no longer needed).
      if (grp.tid == 0) S.n_sort = 0;
      grp.sync();
      for (int b = grp.tid; b < kHashCap; b += nt)
        if (S.hkey[b] != kEmptyKey) {
          const int p = atomicAdd(&S.n_sort, 1);
          S.s1[p] = ~S.hval[b];
          S.s2[p] = S.hkey[b];
        }
      grp.sync();
      const int D = S.n_sort;
      const int npass = min(K, D);  // all hot entries are >= floor
      for (int p = grp.tid; p < D; p += nt) {
        const uint64_t a1 = S.s1[p], a2 = S.s2[p];
        int rk = 0;
        for (int q = 0; q < D; ++q) {
          const uint64_t b1 = S.s1[q], b2 = S.s2[q];
          rk += (b1 < a1 || (b1 == a1 && b2 < a2)) ? 1 : 0;
        }
        if (rk < npass) {
          S.hkey[rk] = a2;
          S.hval[rk] = ~a1;
        }
      }
      if (grp.tid == 0) {
        // max_states beyond the device cap binds when more than kMaxStates
        // distinct keys are at or above the floor: either the hash already
        // holds more, or it holds exactly kMaxStates while candidates in bins
        // past the hot threshold were never scanned.
        if (max_states > kMaxStates && (D > kMaxStates || (D == kMaxStates && S.bstar < kBins)))
          atomicExch(error_flag, 4);
        S.m_first = 0ull;
        S.m_keep = 0ull;
        S.best = best;
        S.floor = floor;
      }
      grp.sync();
      // ---- prune_streams (fsa_search.hpp:240-283) ----
      // In sorted order, the first max_contexts distinct contexts are kept;
      // a passing entry survives iff its context is kept.  Entry p's context
      // is kept iff at most max_contexts distinct contexts appear up to its
      // first occurrence fo: popcount of the first-occurrence mask over
      // [0, fo].  Survivors keep the sorted order (mask prefix counts).
      {
        const int p = grp.tid;
        int fo = p;
        if (p < npass) {
          // first q < p with the same context: a fixed-trip scan (no early
          // exit), so the shared-memory loads pipeline; the lowest match wins
          const int32_t c = static_cast<int32_t>(S.hkey[p] >> 32);
#pragma unroll 8
          for (int q = npass - 1; q >= 0; --q)
            if (q < p && static_cast<int32_t>(S.hkey[q] >> 32) == c) fo = q;
          if (fo == p) atomicOr(&S.m_first, 1ull << p);
        }
        grp.sync();
        const bool keep = p < npass && __popcll(S.m_first & ((2ull << fo) - 1ull)) <= max_contexts;
        if (keep) atomicOr(&S.m_keep, 1ull << p);
        grp.sync();
        if (keep) {
          const int x = __popcll(S.m_keep & ((1ull << p) - 1ull));
          S.surv_ctx[x] = static_cast<int32_t>(S.hkey[p] >> 32);
          S.surv_state[x] = static_cast<int32_t>(S.hkey[p] & 0xffffffffu);
          S.surv_score[x] = dbl_of(S.hval[p]);
        }
        if (p == 0) S.n_surv = __popcll(S.m_keep);
      }
      for (int b = grp.tid; b < kSurvHash; b += nt) S.shkey[b] = kEmptyKey;
      grp.sync();
      // Node ids in (ctx, state) order (274-283): rank among survivors.
      const int nsurv = S.n_surv;
      int my_rank = -1;
      int my_ctx = 0, my_state = 0;
      double my_score = 0;
      if (grp.tid < nsurv) {
        my_ctx = S.surv_ctx[grp.tid];
        my_state = S.surv_state[grp.tid];
        my_score = S.surv_score[grp.tid];
        const uint64_t mk = key_of(my_ctx, my_state);
        int rk = 0;
        for (int z = 0; z < nsurv; ++z) rk += key_of(S.surv_ctx[z], S.surv_state[z]) < mk ? 1 : 0;
        my_rank = rk;
        uint32_t slot = hash_slot(mk, kSurvHash);
        while (atomicCAS(reinterpret_cast<unsigned long long*>(&S.shkey[slot]),
                         static_cast<unsigned long long>(kEmptyKey),
                         static_cast<unsigned long long>(mk)) != kEmptyKey)
          slot = (slot + 1) & (kSurvHash - 1);
        S.shnode[slot] = S.num_nodes + rk;
      }
      grp.sync();
      // ---- lattice arcs: raw candidates into survivors, generation order ----
      FSA_MARK(3);  // rank selection, prune, node ids
      // Pass C: one bit per raw candidate whose key survived.
      for (int q0 = grp.tid; q0 < nraw; q0 += kU * nt) {
        Raw rc[kU];
        bool ok[kU];
        raw_batch(S, q0, nt, nraw, arcs, src, V, rc, ok);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (!ok[u]) continue;
          const uint64_t k = key_of(rc[u].ctx, rc[u].state);
          uint32_t slot = hash_slot(k, kSurvHash);
          while (S.shkey[slot] != kEmptyKey && S.shkey[slot] != k) slot = (slot + 1) & (kSurvHash - 1);
          if (S.shkey[slot] == k) {
            const int q = q0 + u * nt;
            atomicOr(&S.mbits[q >> 5], 1u << (q & 31));
          }
        }
      }
      grp.sync();
      // Each thread owns a contiguous run of bit words, so the scan order is
      // the generation order.
      const int nwords = (nraw + 31) >> 5;
      const int wpt = (nwords + nt - 1) / nt;
      const int w0 = min(nwords, grp.tid * wpt), w1 = min(nwords, w0 + wpt);
      int cnt = 0;
      for (int w = w0; w < w1; ++w) cnt += __popc(S.mbits[w]);
      int total = 0;
      const int my_pos = group_scan(grp, S, cnt, &total);
      if (grp.tid == 0) {
        const unsigned long long off = atomicAdd(lat_count, static_cast<unsigned long long>(total));
        if (static_cast<int64_t>(off + total) > lat_cap) {
          atomicExch(error_flag, 1);  // the host regrows the pool and decodes again
          S.arc_off = -1;
          S.flag |= 2;  // this stream's lattice is incomplete: no best path
        } else {
          S.arc_off = static_cast<int32_t>(off);
        }
        S.arc_count = total;
      }
      grp.sync();
      const int arc_off = S.arc_off;
      if (grp.tid == 0) S.lat_total += total;
      FSA_MARK(4);  // pass C + scan
      // Pass D: only the (few) hits are recomputed and written.
      if (arc_off >= 0) {
        int pos = my_pos;
        for (int w = w0; w < w1; ++w) {
          uint32_t bits = S.mbits[w];
          while (bits) {
            const int q = (w << 5) + __ffs(bits) - 1;
            bits &= bits - 1;
            const Raw rc = raw_cand(S, q, arcs, src, V);
            const uint64_t k = key_of(rc.ctx, rc.state);
            uint32_t slot = hash_slot(k, kSurvHash);
            while (S.shkey[slot] != k) slot = (slot + 1) & (kSurvHash - 1);
            LatArc a;
            a.src = S.act_node[rc.i];
            a.dst = S.shnode[slot];
            a.label = rc.label;
            a.pad = 0;
            a.score = rc.arc_score;
            lat[static_cast<int64_t>(arc_off) + pos++] = a;
          }
        }
      }
      grp.sync();
      FSA_MARK(5);  // pass D
      // New active set, sorted by (ctx, state).
      if (my_rank >= 0) {
        nctx[S.num_nodes + my_rank] = my_ctx;
        S.act_ctx[my_rank] = my_ctx;
        S.act_state[my_rank] = my_state;
        S.act_score[my_rank] = my_score;
        S.act_node[my_rank] = S.num_nodes + my_rank;
      }
      grp.sync();
      if (grp.tid == 0) {
        *finfo_t = make_int4(S.arc_off, S.arc_count, S.num_nodes, nsurv);
        S.n_act = nsurv;
        S.num_nodes += nsurv;
        if (nsurv == 0) S.flag |= 1;  // dead stream (233-238): cannot happen with finite scores
      }
      grp.sync();
}

// lattice_to_best_seq(kMax) = best_path (fsa.hpp:311-376) on the stream's
// HBM lattice, by the first warp of its thread group (lane < 32): backward
// suffix maxima frame by frame (lanes over arcs, shared-memory atomicMax on
// order-preserving bits; layer t+1 in S.act_score, layer t in S.hval, every
// layer also in nb for the trace), then the forward trace taking the first
// arc (lowest index) that attains the remainder (ballot over 32 arcs), next
// frame prefetched.  S.flag / S.num_nodes are the stream's; its other fields
// are scratch.
__device__ __forceinline__ void fsa_best_path(FsaStream& S, int lane, const int4* __restrict__ finfo_s,
                                              const LatArc* __restrict__ lat, double* __restrict__ nb, int32_t T,
                                              int32_t* __restrict__ tokens_s, int32_t* __restrict__ length_s,
                                              double* __restrict__ score_s, int32_t* __restrict__ error_flag) {
    double* cur = S.act_score;                                      // layer t+1 suffix values
    unsigned long long* nxt = reinterpret_cast<unsigned long long*>(S.hval);  // layer t (ordered bits)
    int32_t len = 0;
    double total = 0.0;
    if (!(S.flag & 2)) {
      const int32_t nn = S.num_nodes;
      const int32_t lastb = T > 0 ? finfo_s[T - 1].z : 0;
      for (int32_t n = lastb + lane; n < nn; n += 32) {
        nb[n] = 0.0;  // layer T reaches the super-final node by a score-0 arc
        cur[n - lastb] = 0.0;
      }
      __syncwarp();
      // frame t-1's info and first 32 arcs are loaded while frame t is reduced
      int4 fi_p = T > 0 ? finfo_s[T - 1] : make_int4(0, 0, 0, 0);
      LatArc e_p{};
      if (T > 0 && lane < fi_p.y) e_p = lat[static_cast<int64_t>(fi_p.x) + lane];
      for (int32_t t = T - 1; t >= 0; --t) {
        const int4 fi = fi_p;
        const LatArc e0 = e_p;
        if (t > 0) {
          fi_p = finfo_s[t - 1];
          if (lane < fi_p.y) e_p = lat[static_cast<int64_t>(fi_p.x) + lane];
        }
        const int32_t lb = t > 0 ? fi_p.z : 0;
        const int32_t ln = t > 0 ? fi_p.w : 1;
        for (int32_t i = lane; i < ln; i += 32) nxt[i] = 0ull;  // below ord_of(-inf)
        __syncwarp();
        for (int32_t a = lane; a < fi.y; a += 32) {
          const LatArc e = a < 32 ? e0 : lat[static_cast<int64_t>(fi.x) + a];
          atomicMax(&nxt[e.src - lb], ord_of(e.score + cur[e.dst - fi.z]));
        }
        __syncwarp();
        for (int32_t i = lane; i < ln; i += 32) {
          const double v = nxt[i] ? dbl_of(nxt[i]) : -INFINITY;
          cur[i] = v;
          nb[lb + i] = v;
        }
        __syncwarp();
      }
      double remaining = T > 0 ? nb[0] : 0.0;
      if (remaining == -INFINITY || S.flag) {
        total = -INFINITY;
      } else {
        int32_t n = 0;
        LatArc e_n{};
        double v_n = 0.0;
        int4 fi_n = T > 0 ? finfo_s[0] : make_int4(0, 0, 0, 0);
        if (T > 0 && lane < fi_n.y) {
          e_n = lat[static_cast<int64_t>(fi_n.x) + lane];
          v_n = nb[e_n.dst];
        }
        for (int32_t t = 0; t < T; ++t) {
          const int4 fi = fi_n;
          const LatArc e0 = e_n;
          const double v0 = v_n;
          if (t + 1 < T) {  // prefetch frame t+1's first 32 arcs and their suffix values
            fi_n = finfo_s[t + 1];
            if (lane < fi_n.y) {
              e_n = lat[static_cast<int64_t>(fi_n.x) + lane];
              v_n = nb[e_n.dst];
            }
          }
          int32_t chosen = -1;
          LatArc ce{};
          for (int32_t a0 = 0; a0 < fi.y && chosen < 0; a0 += 32) {
            LatArc e = e0;
            double v = v0;
            if (a0 > 0 && a0 + lane < fi.y) {
              e = lat[static_cast<int64_t>(fi.x) + a0 + lane];
              v = nb[e.dst];
            }
            const bool hit = a0 + lane < fi.y && e.src == n && e.score + v == remaining;
            const unsigned ball = __ballot_sync(0xffffffffu, hit);
            if (ball) {
              const int src_lane = __ffs(ball) - 1;
              chosen = a0 + src_lane;
              ce.dst = __shfl_sync(0xffffffffu, e.dst, src_lane);
              ce.label = __shfl_sync(0xffffffffu, e.label, src_lane);
              ce.score = __shfl_sync(0xffffffffu, e.score, src_lane);
              remaining = __shfl_sync(0xffffffffu, v, src_lane);
            }
          }
          if (chosen < 0) {  // best_path "inconsistent scores"
            if (lane == 0) atomicExch(error_flag, 5);
            break;
          }
          if (ce.label != 0) {
            if (lane == 0) tokens_s[len] = ce.label;
            ++len;
          }
          total += ce.score;
          n = ce.dst;
        }
        total += 0.0;  // the score-0 hop into the super-final node
        total += 0.0;  // its final score
      }
    }
    if (lane == 0) {
      *length_s = len;
      *score_s = (S.flag & 2) ? 0.0 : total;
    }
  }

__global__ void __launch_bounds__(kDecodeThreads, 1)
    fsa_kernel(ModelView m, const float* __restrict__ pe, const int32_t* __restrict__ frame_splits,
               int32_t B, int32_t G, int32_t bk, const ArcRec* __restrict__ arcs,
               const int32_t* __restrict__ gsplits, const double* __restrict__ gmaxw,
               double beam, int32_t max_states,
               int32_t max_contexts, LatArc* __restrict__ lat, int64_t lat_cap,
               unsigned long long* __restrict__ lat_count, int4* __restrict__ finfo,
               double* __restrict__ nodebest, int32_t* __restrict__ node_ctx, int32_t* __restrict__ tokens,
               int32_t* __restrict__ lengths, double* __restrict__ scores,
               unsigned long long* __restrict__ counters, int32_t* __restrict__ error_flag) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* HL = reinterpret_cast<float*>(smem_raw);
  const int hl_floats = hl_floats_of(m.J, m.Vp);
  float* W0 = HL + hl_floats;
  float* W1 = W0 + bk * m.Vp;
  FsaSmem& C = *reinterpret_cast<FsaSmem*>(W1 + bk * m.Vp);
  FsaStream* SS = reinterpret_cast<FsaStream*>(&C + 1);

  const int s0 = blockIdx.x * G;
  const int ns = min(G, B - s0);
  if (ns <= 0) return;
  const WPipe& pipe = C.pipe;
  const int nt = kDecodeThreads / G;
  const Group grp{static_cast<int>(threadIdx.x) / nt, static_cast<int>(threadIdx.x) % nt, nt};
  const bool have = grp.id < ns;
  FsaStream& S = SS[grp.id < ns ? grp.id : 0];
  const int sidx = s0 + grp.id;
  const int32_t fs = have ? frame_splits[sidx] : 0;
  const int32_t T = have ? frame_splits[sidx + 1] - fs : 0;
  const int K = min(max_states, kMaxStates);
  const int64_t fbase = static_cast<int64_t>(fs) + sidx;          // frame info base
  const int64_t nbase = static_cast<int64_t>(fs) * K + sidx;       // node-best base
  // Histogram range below the upper bound: the beam (capped at 8 nats) plus
  // 2 nats of slack for the gap between the bound and the true best.
  const double scale = kBins / ((beam < 8.0 ? beam : 8.0) + 2.0);
  const int M = K + 32;  // hot-candidate target

  int32_t tmax = 0;
  for (int i = 0; i < ns; ++i) tmax = max(tmax, frame_splits[s0 + i + 1] - frame_splits[s0 + i]);
  if (have && grp.tid == 0) {  // init_streams (95-120): ((0,0), state 0, 0.0, node 0)
    node_ctx[nbase] = 0;
    S.n_act = 1;
    S.num_nodes = 1;
    S.act_ctx[0] = 0;
    S.act_state[0] = 0;
    S.act_score[0] = 0.0;
    S.act_node[0] = 0;
    S.flag = 0;
  }
  if (threadIdx.x == 0) {
    C.pipe = make_wpipe(W0, W1, C.bar, C.wcur, m, bk);
    C.rows_total = 0;
    C.ph[0] = C.ph[1] = C.ph[2] = 0;
    mbar_init(&C.bar[0], 1);
    mbar_init(&C.bar[1], 1);
    fence_mbar_init();
  }
  if (have && grp.tid == 0) S.raw_total = S.lat_total = 0;
#if RNNTG_FSA_PASS_CLOCKS
  if (have && grp.tid == 0)
    for (int i = 0; i < 8; ++i) S.pclk[i] = 0;
#endif
  load_exp_table(C.etab);
  __syncthreads();
  if (threadIdx.x == 0) {
    wpipe_issue(pipe, m, 0);
    wpipe_issue(pipe, m, 1);
  }
  uint32_t gch = 0;

  for (int32_t t = 0; t < tmax; ++t) {
    const bool live = have && t < T;
    // get_contexts: distinct contexts in order; each tuple's row.
    if (live && grp.tid == 0) {
      int nr = 0;
      for (int i = 0; i < S.n_act; ++i) {
        if (nr == 0 || S.row_ctx[nr - 1] != S.act_ctx[i]) S.row_ctx[nr++] = S.act_ctx[i];
        S.act_row[i] = nr - 1;
      }
      S.nrows = nr;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int R = 0;
      for (int g2 = 0; g2 < ns; ++g2) {
        FsaStream& X = SS[g2];
        const int32_t f2 = frame_splits[s0 + g2];
        if (t >= frame_splits[s0 + g2 + 1] - f2) continue;
        X.row_base = R;
        for (int r = 0; r < X.nrows; ++r) {
          if (R < kRowCap) {
            C.row_pe[R] = f2 + t;
            C.row_ctx[R] = X.row_ctx[r];
          }
          ++R;
        }
      }
      if (R > kRowCap) {
        atomicExch(error_flag, 2);  // more joiner rows than the CTA tile holds
        R = kRowCap;
      }
      C.nrows = R;
      // the exact log-softmax borrows the weight stages when its scratch fits
      C.pipe.defer = (C.pipe.nc >= 2 && lse_cta_fits(R, m.V, bk * m.Vp)) ? 1 : 0;
    }
    __syncthreads();
    const int R = C.nrows;
    if (threadIdx.x == 0) C.rows_total += R;
    const long long c0 = clock64();
    build_h(m, pe, C.row_pe, C.row_ctx, R, HL);
    const long long c1 = clock64();
    joiner_gemm(m, pipe, gch, HL, R);
    const long long c2 = clock64();
    if (pipe.defer) {  // CTA-wide exact normalisers in the weight stages
      double* E = reinterpret_cast<double*>(W0);
      lse_cta_exps(HL, E, bk * m.Vp, m.Vp, m.V, R, C.etab, C.row_m);
      if (threadIdx.x < 32) {
        lse_cta_chain(HL, E, bk * m.Vp, m.Vp, m.V, R, C.row_m, C.row_lse, nullptr);
        if (threadIdx.x < R) C.row_lpmax[threadIdx.x] = static_cast<double>(C.row_m[threadIdx.x]) - C.row_lse[threadIdx.x];
      }
      __syncthreads();
      wpipe_issue_next(pipe, m, gch);
    } else {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int r = warp; r < R; r += kDecodeThreads / 32) {
        const float* L = HL + static_cast<int64_t>(r) * m.Vp;
        const double lse = row_lse(L, m.V, lse_scratch(HL, m.Vp), C.etab);
        float mx = -FLT_MAX;
        for (int k = lane; k < m.V; k += 32) mx = fmaxf(mx, L[k]);
        mx = warp_max_f(mx);
        if (lane == 0) {
          C.row_lse[r] = lse;
          C.row_lpmax[r] = static_cast<double>(mx) - lse;
        }
      }
    }
    __syncthreads();

#if RNNTG_FSA_PASS_CLOCKS
    if (live && grp.tid == 0) S.pclk_last = clock64();
#endif
    if (live)
      fsa_frame(S, grp, LpJoiner{HL, C.row_lse, m.Vp}, C.row_lpmax, m.V, arcs, gsplits, gmaxw, beam, K, max_states,
                max_contexts, M, scale, lat, lat_cap, lat_count, finfo + fbase + t, node_ctx + nbase, error_flag);
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long c4 = clock64();
      C.ph[0] += c1 - c0;
      C.ph[1] += c2 - c1;
      C.ph[2] += c4 - c2;
    }
  }

  // ---- lattice_to_best_seq(kMax) = best_path on the stream's lattice ----
  // (fsa.hpp:311-376) by the group's first warp.  Backward: frame by frame,
  // suffix maxima of the layer-t nodes from their arcs (lanes over arcs,
  // shared-memory atomicMax on order-preserving bits: max is order
  // independent), layer t+1's values in shared memory, every layer also in
  // HBM for the trace.  Forward: from node 0, the first arc (lowest index)
  // attaining the remainder -- lanes test 32 arcs at once, ballot, first set
  // bit -- with the next frame's arcs and suffix values loaded while this
  // frame's choice is made.
  const long long cb0 = clock64();
  __syncthreads();  // the frame loop's shared state is free from here on
  if (have && grp.tid < 32)
    fsa_best_path(S, grp.tid, finfo + fbase, lat, nodebest + nbase, T, tokens + fs, lengths + sidx, scores + sidx,
                  error_flag);
  if (grp.tid == 0 && have) atomicAdd(&counters[11], static_cast<unsigned long long>(clock64() - cb0));
  if (threadIdx.x == 0) {
    atomicAdd(&counters[8], static_cast<unsigned long long>(C.ph[0]));
    atomicAdd(&counters[9], static_cast<unsigned long long>(C.ph[1]));
    atomicAdd(&counters[10], static_cast<unsigned long long>(C.ph[2]));
    mbar_wait(&C.bar[gch & 1u], (gch >> 1) & 1u);
    mbar_wait(&C.bar[(gch + 1) & 1u], ((gch + 1) >> 1) & 1u);
    unsigned long long sf = 0;
    for (int i = 0; i < ns; ++i) sf += frame_splits[s0 + i + 1] - frame_splits[s0 + i];
    atomicAdd(&counters[0], sf);
    atomicAdd(&counters[1], C.rows_total);
  }
  if (have && grp.tid == 0) {
    atomicAdd(&counters[2], S.raw_total);
#if RNNTG_FSA_PASS_CLOCKS
    if (grp.id == 0) {  // development: setup + pass A | pass B + prune | pass C + D
      atomicAdd(&counters[5], static_cast<unsigned long long>(S.pclk[0] + S.pclk[1]));
      atomicAdd(&counters[6], static_cast<unsigned long long>(S.pclk[2] + S.pclk[3]));
      atomicAdd(&counters[7], static_cast<unsigned long long>(S.pclk[4] + S.pclk[5]));
    }
#endif
    atomicAdd(&counters[3], S.lat_total);
  }
}

// ---------------------------------------------------------------------------
// The Algorithm-1 step API (fsa_search.hpp:95-297, Algorithm 1):
// the caller runs its own model between get_contexts and expand_arcs and
// hands the log-prob rows in; the decoder's expand / prune (fsa_frame with
// LpRows) and best path run on the GPU.  Stream state lives in HBM between
// steps (StepState, the reference's DecodeStream minus the host vectors).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kDecodeThreads, 1) fsa_step_kernel(FsaStepArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int G = a.G;
  FsaStream* SS = reinterpret_cast<FsaStream*>(smem_raw);
  double* lpmax_all = reinterpret_cast<double*>(SS + G);  // [G][kMaxStates]
  const int s0 = blockIdx.x * G;
  const int ns = min(G, a.B - s0);
  const int nt = kDecodeThreads / G;
  const Group grp{static_cast<int>(threadIdx.x) / nt, static_cast<int>(threadIdx.x) % nt, nt};
  const bool have = grp.id < ns;
  if (!have) return;  // whole groups only: named barriers are per group
  FsaStream& S = SS[grp.id];
  double* lpmax = lpmax_all + grp.id * kMaxStates;
  const int sidx = s0 + grp.id;
  FsaStepState& X = static_cast<FsaStepState*>(a.state)[sidx];
  const int32_t fs = a.frame_splits[sidx];
  const int K = min(a.max_states, kMaxStates);
  const int64_t fbase = static_cast<int64_t>(fs) + sidx;
  const int64_t nbase = static_cast<int64_t>(fs) * K + sidx;
  const int32_t t = X.t, T = X.T;
  if (t >= T) return;  // done (finish_stream at its last frame)
  if (grp.tid == 0) {
    S.n_act = X.n_act;
    S.num_nodes = X.num_nodes;
    S.flag = X.flag;
    S.raw_total = S.lat_total = 0;
    if (t == 0) a.node_ctx[nbase] = 0;
  }
  grp.sync();
  for (int i = grp.tid; i < S.n_act; i += nt) {
    S.act_ctx[i] = X.act_ctx[i];
    S.act_state[i] = X.act_state[i];
    S.act_score[i] = X.act_score[i];
    S.act_node[i] = X.act_node[i];
  }
  grp.sync();
  // get_contexts (124-154): the caller's rows for this stream must be its
  // distinct active contexts in order (else "stale get_contexts data")
  if (grp.tid == 0) {
    int nr = 0;
    for (int i = 0; i < S.n_act; ++i) {
      if (nr == 0 || S.row_ctx[nr - 1] != S.act_ctx[i]) S.row_ctx[nr++] = S.act_ctx[i];
      S.act_row[i] = nr - 1;
    }
    S.nrows = nr;
    S.row_base = a.row_splits[sidx];
    if (a.row_splits[sidx + 1] - S.row_base != nr) atomicExch(a.error_flag, 7);
  }
  grp.sync();
  if (a.row_splits[sidx + 1] - S.row_base != S.nrows) return;
  // row maxima of the caller's rows (the frame's upper bound, fsa_frame)
  for (int r = 0; r < S.nrows; ++r) {
    const double* P = a.P + static_cast<int64_t>(S.row_base + r) * a.V;
    double mx = -INFINITY;
    for (int k = grp.tid; k < a.V; k += nt) mx = fmax(mx, P[k]);
    mx = group_max(grp, S, mx);
    if (grp.tid == 0) lpmax[r] = mx;
  }
  grp.sync();
  const double scale = kBins / ((a.beam < 8.0 ? a.beam : 8.0) + 2.0);
  fsa_frame(S, grp, LpRows{a.P, a.V}, lpmax - S.row_base, a.V, static_cast<const ArcRec*>(a.graph_arcs),
            a.graph_splits, a.graph_maxw, a.beam, K, a.max_states, a.max_contexts, K + 32, scale,
            static_cast<LatArc*>(a.lattice), a.lattice_cap, a.lattice_count,
            reinterpret_cast<int4*>(a.lat_frame_info) + fbase + t, a.node_ctx + nbase, a.error_flag);
  // back to HBM
  for (int i = grp.tid; i < S.n_act; i += nt) {
    X.act_ctx[i] = S.act_ctx[i];
    X.act_state[i] = S.act_state[i];
    X.act_score[i] = S.act_score[i];
    X.act_node[i] = S.act_node[i];
  }
  if (grp.tid == 0) {
    X.n_act = S.n_act;
    X.num_nodes = S.num_nodes;
    X.flag = S.flag;
    X.t = t + 1;
    atomicAdd(&a.counters[2], S.raw_total);
    atomicAdd(&a.counters[3], S.lat_total);
    atomicAdd(&a.counters[0], 1ull);
  }
}

// finish_stream + lattice_to_best_seq(kMax) of every stream (the driver's
// tail, fsa_search.hpp:375-387).
__global__ void __launch_bounds__(kDecodeThreads, 1) fsa_step_finish_kernel(FsaStepArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int G = a.G;
  FsaStream* SS = reinterpret_cast<FsaStream*>(smem_raw);
  const int s0 = blockIdx.x * G;
  const int ns = min(G, a.B - s0);
  const int nt = kDecodeThreads / G;
  const Group grp{static_cast<int>(threadIdx.x) / nt, static_cast<int>(threadIdx.x) % nt, nt};
  if (grp.id >= ns) return;
  FsaStream& S = SS[grp.id];
  const int sidx = s0 + grp.id;
  const FsaStepState& X = static_cast<const FsaStepState*>(a.state)[sidx];
  const int32_t fs = a.frame_splits[sidx];
  const int32_t T = a.frame_splits[sidx + 1] - fs;
  const int K = min(a.max_states, kMaxStates);
  const int64_t nbase = static_cast<int64_t>(fs) * K + sidx;
  if (grp.tid == 0) {
    S.flag = X.flag | (X.t < T ? 4 : 0);  // a stream stopped before its last frame has no complete path
    S.num_nodes = X.num_nodes;
    if (T == 0) a.node_ctx[nbase] = 0;
  }
  grp.sync();
  if (grp.tid < 32)
    fsa_best_path(S, grp.tid, reinterpret_cast<const int4*>(a.lat_frame_info) + fs + sidx,
                  static_cast<const LatArc*>(a.lattice), a.node_best + nbase, T, a.tokens + fs, a.lengths + sidx,
                  a.scores + sidx, a.error_flag);
}

}  // namespace

size_t fsa_stream_smem() { return sizeof(FsaStream); }

static int step_streams_per_cta(int K) { return K > 16 ? 2 : 4; }

cudaError_t launch_fsa_step(FsaStepArgs a, bool finish, cudaStream_t s) {
  if (a.B <= 0) return cudaSuccess;
  const int K = std::min(a.max_states, kMaxStates);
  a.G = step_streams_per_cta(K);
  const size_t smem = sizeof(FsaStream) * a.G + (finish ? 0 : sizeof(double) * kMaxStates * a.G);
  auto kern = finish ? fsa_step_finish_kernel : fsa_step_kernel;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<(a.B + a.G - 1) / a.G, kDecodeThreads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_decode_fsa(const DecodeArgs& a, cudaStream_t s) {
  const ModelView m = view_of(*a.m);
  const int G = a.streams_per_cta;
  // 32-row weight chunks when they fit beside G stream states, else 16.
  int max_smem = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t rest = sizeof(FsaSmem) + sizeof(FsaStream) * G;
  const int bk = smem_common(m, kBK) + rest <= static_cast<size_t>(max_smem) ? kBK : kBKSmall;
  const size_t smem = smem_common(m, bk) + rest;
  cudaError_t e = cudaFuncSetAttribute(fsa_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int grid = (a.B + G - 1) / G;
  fsa_kernel<<<grid, kDecodeThreads, smem, s>>>(
      m, a.pe, a.frame_splits, a.B, G, bk, static_cast<const ArcRec*>(a.graph_arcs), a.graph_splits,
      a.graph_maxw, a.fsa_beam, a.max_states, a.max_contexts, static_cast<LatArc*>(a.lattice), a.lattice_cap,
      a.lattice_count, reinterpret_cast<int4*>(a.lat_frame_info), a.node_best, a.node_ctx, a.tokens, a.lengths,
      a.scores, a.counters, a.error_flag);
  return cudaGetLastError();
}

}  // namespace rnntg
