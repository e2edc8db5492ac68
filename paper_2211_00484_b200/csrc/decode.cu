// Persistent, stream-stationary decode kernels (greedy / modified beam).
//
// One CTA owns a fixed group of G streams for the whole utterance and loops
// over frames itself: streams are independent (batching transparency,
// search_test.cpp:169-187, fsa_search_test.cpp:364-393), so no grid-wide
// synchronisation and no per-frame kernel launch exists.  Per frame the CTA
//
//   A. lists its joiner rows: one per distinct (stream, packed context) —
//      rows are a pure function of (stream, frame, context) (model.hpp:240),
//      so hypotheses sharing a context share a row, bit-identically;
//   B. builds h[r] = tanhf((pe + pd[ctx]) + j_b) in shared memory
//      (joiner_logits_from_proj, model.hpp:284-292; pd from the K0 table);
//   C. computes logits = out_b + out_w . h with sequential non-fused fp32 on
//      CUDA cores, out_w streamed from L2 in 32 KB k-chunks by
//      cp.async.bulk + mbarrier (double buffered, prefetching across frame
//      boundaries because the chunk sequence is data independent);
//   D. reduces each row: greedy first-max argmax (search.hpp:59-66); beam
//      log-softmax normaliser (model.hpp:115-125) and the row's top-B tokens;
//   E. advances each stream's search state (warp per stream).
//
// After the last frame a warp per stream traces the back-pointer lattice
// (kept in HBM) and writes the token sequence.
#include <float.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "decode_common.cuh"

namespace rnntg {
namespace {

using namespace dec;

// ---------------------------------------------------------------------------
// Greedy.  cap = 1: greedy_search_batch (search.hpp:107-167, S = 1).  cap > 1:
// greedy_search (search.hpp:76-100) per stream — on a frame, repeat
// {joiner, first-max argmax} until blank or `cap` emissions, each emission
// advancing the context; every sub-step is one GEMM pass over the streams
// still open on the frame.  Stream i's tokens go to its slot region
// [cap * frame_splits[i], cap * frame_splits[i+1]).
// ---------------------------------------------------------------------------
struct GreedySmem {
  uint64_t bar[2];
  uint32_t wcur[2];
  int64_t row_pe[kRowCap];
  int32_t row_ctx[kRowCap];
  int32_t row_stream[kRowCap];
  int32_t ctx[kRowCap];
  int32_t len[kRowCap];
  int32_t open[kRowCap];
  int32_t capped;
  int32_t nrows;
};

__global__ void __launch_bounds__(kDecodeThreads, 1)
    greedy_kernel(ModelView m, const float* __restrict__ pe,
                  const int32_t* __restrict__ frame_splits, int32_t B,
                  int32_t G, int32_t cap, int32_t count_capped, int32_t* __restrict__ tokens,
                  int32_t* __restrict__ lengths,
                  unsigned long long* __restrict__ counters) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* HL = reinterpret_cast<float*>(smem_raw);
  const int hl_floats = hl_floats_of(m.J, m.Vp);
  float* W0 = HL + hl_floats;
  float* W1 = W0 + kBK * m.Vp;
  GreedySmem& S = *reinterpret_cast<GreedySmem*>(W1 + kBK * m.Vp);

  const int s0 = blockIdx.x * G;
  const int ns = min(G, B - s0);
  if (ns <= 0) return;
  WPipe pipe = make_wpipe(W0, W1, S.bar, S.wcur, m);

  int32_t tmax = 0;
  for (int i = 0; i < ns; ++i)
    tmax = max(tmax, frame_splits[s0 + i + 1] - frame_splits[s0 + i]);
  if (threadIdx.x < ns) {
    S.ctx[threadIdx.x] = 0;
    S.len[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) {
    S.capped = 0;
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    wpipe_issue(pipe, m, 0);
    wpipe_issue(pipe, m, 1);
  }
  uint32_t g = 0;
  unsigned long long rows_total = 0;

  for (int32_t t = 0; t < tmax; ++t) {
    if (threadIdx.x < ns) {
      const int32_t fs = frame_splits[s0 + threadIdx.x];
      S.open[threadIdx.x] = t < frame_splits[s0 + threadIdx.x + 1] - fs;
    }
    for (int32_t n = 0; n < cap; ++n) {
      __syncthreads();
      if (threadIdx.x == 0) {  // A. one row per stream still open on the frame
        int R = 0;
        for (int i = 0; i < ns; ++i) {
          if (!S.open[i]) continue;
          S.row_pe[R] = frame_splits[s0 + i] + t;
          S.row_ctx[R] = S.ctx[i];
          S.row_stream[R] = i;
          ++R;
        }
        S.nrows = R;
      }
      __syncthreads();
      const int R = S.nrows;
      if (R == 0) break;  // CTA-uniform
      rows_total += R;
      build_h(m, pe, S.row_pe, S.row_ctx, R, HL);
      joiner_gemm(m, pipe, g, HL, R);
      // D+E. first-max argmax of the raw float logits (search.hpp:59-66);
      // blank closes the stream's frame, a token advances its context.
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int r = warp; r < R; r += kWarps) {
        const float* L = HL + static_cast<int64_t>(r) * m.Vp;
        float bv = -FLT_MAX;
        int bk = 0x7fffffff;
        for (int k = lane; k < m.V; k += 32)
          if (tok_before(L[k], k, bv, bk)) {
            bv = L[k];
            bk = k;
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
          if (tok_before(ov, ok, bv, bk)) {
            bv = ov;
            bk = ok;
          }
        }
        if (lane == 0) {
          const int i = S.row_stream[r];
          if (bk == 0) {
            S.open[i] = 0;
          } else {
            const int32_t len = S.len[i];
            tokens[static_cast<int64_t>(cap) * frame_splits[s0 + i] + len] = bk;
            S.len[i] = len + 1;
            S.ctx[i] = (S.ctx[i] % m.V) * m.V + bk;
            if (n + 1 == cap && count_capped) atomicAdd(&S.capped, 1);
          }
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < ns) lengths[s0 + threadIdx.x] = S.len[threadIdx.x];
  // Drain the two prefetched chunks before the CTA's smem is released.
  if (threadIdx.x == 0) {
    mbar_wait(&S.bar[g & 1u], (g >> 1) & 1u);
    mbar_wait(&S.bar[(g + 1) & 1u], ((g + 1) >> 1) & 1u);
    unsigned long long sf = 0;
    for (int i = 0; i < ns; ++i) sf += frame_splits[s0 + i + 1] - frame_splits[s0 + i];
    atomicAdd(&counters[0], sf);
    atomicAdd(&counters[1], rows_total);
    if (S.capped) atomicAdd(&counters[13], static_cast<unsigned long long>(S.capped));
  }
}

// ---------------------------------------------------------------------------
// Modified beam search (beam_search at max_symbols = 1, search.hpp:206-277).
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}
// Sequence identity: two independent chained 64-bit hashes of ys plus
// |ys| and the last token.
__device__ __forceinline__ uint64_t hash_ext1(uint64_t h, int32_t k) {
  return mix64(h + 0x9e3779b97f4a7c15ull * static_cast<uint64_t>(k + 1));
}
__device__ __forceinline__ uint64_t hash_ext2(uint64_t h, int32_t k) {
  return mix64((h ^ 0xd6e8feb86659fd93ull) * 0x100000001b3ull +
               static_cast<uint64_t>(k) * 0xff51afd7ed558ccdull);
}

struct Hyps {  // one stream's beam, sorted best first
  double score[kMaxBeam];
  uint64_t h1[kMaxBeam], h2[kMaxBeam], p1[kMaxBeam], p2[kMaxBeam];
  int32_t ctx[kMaxBeam], len[kMaxBeam], last[kMaxBeam], row[kMaxBeam];
  int32_t nh;
};

// Time-sliced launches (DecodeArgs::t0/t1): frames [t0, t1) of every stream;
// the hypothesis sets are loaded from / stored to `state` (indexed by stream)
// at the launch boundaries.  t0 = 0, t1 = INT_MAX, state = nullptr: one
// launch over all frames.
struct BeamSlice {
  int32_t t0, t1;
  Hyps* state;
};
static_assert(sizeof(Hyps) % 8 == 0, "hypothesis sets are copied as 8-byte words");

// CTA-wide copy of n hypothesis sets (out of line: keeps the frame loop's
// register allocation independent of the slice plumbing).
__device__ __noinline__ void copy_hyps(Hyps* __restrict__ dst, const Hyps* __restrict__ src, int n) {
  constexpr int W = sizeof(Hyps) / 8;
  uint64_t* d = reinterpret_cast<uint64_t*>(dst);
  const uint64_t* s = reinterpret_cast<const uint64_t*>(src);
  for (int x = threadIdx.x; x < n * W; x += blockDim.x) d[x] = s[x];
}

struct BeamCand {  // stage-1 extension or stage-2 merged entry
  double score;
  uint64_t h1, h2, p1, p2;
  int32_t parent;  // hypothesis slot at layer t
  int32_t tok;     // 0 = blank continuation (the parent's own ys)
  int32_t len, ctx, last;
};

struct BeamSmem {
  uint64_t etab[256];  // glibc exp table (lse_exact)
  float row_m[kRowCap];  // row maxima (beam_reduce_cta)
  unsigned long long stat[16];  // per-CTA counters (layout of DecodeArgs::counters)
  WPipe pipe;
  uint64_t bar[2];
  uint32_t wcur[2];
  int64_t row_pe[kRowCap];
  int32_t row_ctx[kRowCap];
  double row_lse[kRowCap];
  float row_l0[kRowCap];
  float row_tl[kRowCap][kMaxBeam];
  int32_t row_tk[kRowCap][kMaxBeam];
  int32_t nrows;
};

struct TcBars {  // tcgen05 variant: stage and completion barriers, TMEM base
  uint64_t full[kTcStages], empty[kTcStages], done;
  uint32_t tmem_addr;
};

// Walks two equal-length sequences backwards through the back-pointer
// lattice and returns <0, 0, >0 for lexicographic X<Y, X==Y, X>Y.  Each
// sequence is (layer tau, slot, pending token or -1).  Only reached on exact
// score ties (the third key of hyp_better, search.hpp:172-178).
__device__ int lex_cmp(const uint32_t* __restrict__ bp, int tx, int sx, int px,
                       int ty, int sy, int py) {
  int res = 0;
  while (true) {
    if (px < 0 && py < 0 && tx == ty && sx == sy) break;  // shared prefix
    int a = -1, b = -1;
    if (px >= 0) {
      a = px;
      px = -1;
    } else {
      while (tx > 0) {
        const uint32_t e = bp[tx * kMaxBeam + sx];
        --tx;
        sx = static_cast<int>(e & 0xffu);
        const int tok = static_cast<int>(e >> 8);
        if (tok != 0) {
          a = tok;
          break;
        }
      }
    }
    if (py >= 0) {
      b = py;
      py = -1;
    } else {
      while (ty > 0) {
        const uint32_t e = bp[ty * kMaxBeam + sy];
        --ty;
        sy = static_cast<int>(e & 0xffu);
        const int tok = static_cast<int>(e >> 8);
        if (tok != 0) {
          b = tok;
          break;
        }
      }
    }
    if (a < 0 || b < 0) break;
    if (a != b) res = a < b ? -1 : 1;
  }
  return res;
}

// hyp_better(a, b) over candidates of one frame (search.hpp:172-178).
__device__ __forceinline__ bool cand_before(const BeamCand& a, double ka,
                                            const BeamCand& b, double kb,
                                            const uint32_t* bp, int layer,
                                            unsigned long long* ties) {
  if (ka != kb) return ka > kb;
  if (a.len != b.len) return a.len < b.len;
  ++*ties;
  // Same length.  Extensions of the same parent: smaller token first.
  if (a.tok != 0 && b.tok != 0 && a.parent == b.parent) return a.tok < b.tok;
  const int c = lex_cmp(bp, layer, a.parent, a.tok != 0 ? a.tok : -1, layer,
                        b.parent, b.tok != 0 ? b.tok : -1);
  return c < 0;
}

// Per-row results of the row reduction, consumed by the beam step.
struct RowRes {
  double* lse;
  float* l0;
  float (*tl)[kMaxBeam];
  int32_t (*tk)[kMaxBeam];
};

// A. joiner rows for n streams (one warp, lane = stream): one row per
// distinct context among a live stream's hypotheses; writes the row tables
// and each hypothesis' row index.  Returns the row count (warp-uniform).
__device__ __forceinline__ int beam_rows(Hyps* H, int n, const int32_t* fsp, int t,
                                         int64_t* row_pe, int32_t* row_ctx) {
  const int lane = threadIdx.x & 31;
  const int i = lane;
  int cnt = 0;
  if (i < n && t < fsp[i + 1] - fsp[i]) {
    const Hyps& h = H[i];
    for (int j = 0; j < h.nh; ++j) {
      bool fresh = true;
      for (int q = 0; q < j; ++q) fresh = fresh && h.ctx[q] != h.ctx[j];
      cnt += fresh ? 1 : 0;
    }
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (cnt > 0) {
    Hyps& h = H[i];
    const int64_t pr = fsp[i] + t;
    int r = incl - cnt;
    for (int j = 0; j < h.nh; ++j) {
      int first = j;
      for (int q = j - 1; q >= 0; --q)
        if (h.ctx[q] == h.ctx[j]) first = q;
      if (first == j) {
        row_pe[r] = pr;
        row_ctx[r] = h.ctx[j];
        h.row[j] = r++;
      } else {
        h.row[j] = h.row[first];
      }
    }
  }
  return __shfl_sync(0xffffffffu, incl, 31);
}

// D for NR rows per warp (rows r0 + 16 j), their dependency chains
// interleaved.  Per row: each lane keeps a sorted top-BCAP of its columns
// k >= 1 (k = lane + 32 i) as 64-bit keys (ordered logit << 32 | ~k: key
// order is (logit desc, token asc)) by branch-free compare-exchange; `beam`
// pops take the warp maximum with two redux.sync each; the row max M is the
// larger of the first pop and the blank logit; then the exact lse
// (lse_exact: the reference's index-order sum with glibc exp / log).
__device__ __forceinline__ uint64_t tok_key(float v, int k) {
  return (static_cast<uint64_t>(ord_key(v + 0.0f)) << 32) | static_cast<uint32_t>(~k);  // -0 -> +0
}

#ifndef RNNTG_TOPK_UNROLL
#define RNNTG_TOPK_UNROLL 2  // 0: compiler's choice
#endif
constexpr int kTopkUnroll = RNNTG_TOPK_UNROLL > 0 ? RNNTG_TOPK_UNROLL : 1;
#ifndef RNNTG_MAIN_STEP_NI
#define RNNTG_MAIN_STEP_NI 0
#endif
#ifndef RNNTG_MAIN_RR_NI
#define RNNTG_MAIN_RR_NI 0
#endif
#ifndef RNNTG_SL_STEP_NI
#define RNNTG_SL_STEP_NI 1
#endif
#ifndef RNNTG_SL_RR_NI
#define RNNTG_SL_RR_NI 1
#endif
template <int BCAP, int NR, bool LSE = true>
__device__ __forceinline__ void beam_row_reduce_n(float* HL, int Vp, int V, int beam, int r0,
                                                  int R, RowRes rr, const uint64_t* etab, int rs = 16) {
  const int lane = threadIdx.x & 31;
  uint64_t t[NR][BCAP];
  const float* L[NR];
  bool live[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    live[j] = r0 + rs * j < R;
    L[j] = HL + static_cast<int64_t>(live[j] ? r0 + rs * j : r0) * Vp;
#pragma unroll
    for (int q = 0; q < BCAP; ++q) t[j][q] = 0;
  }
#if RNNTG_TOPK_UNROLL > 0
#pragma unroll kTopkUnroll
#endif
  for (int k = lane; k < V; k += 32) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      uint64_t c = k >= 1 ? tok_key(L[j][k], k) : 0;
#pragma unroll
      for (int q = 0; q < BCAP; ++q) {
        const uint64_t hi = max(t[j][q], c);
        c = min(t[j][q], c);
        t[j][q] = hi;
      }
    }
  }
  float M[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) M[j] = L[j][0];
  for (int q = 0; q < beam; ++q) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const uint32_t H = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(t[j][0] >> 32));
      const uint32_t Lo = __reduce_max_sync(
          0xffffffffu, static_cast<uint32_t>(t[j][0] >> 32) == H ? static_cast<uint32_t>(t[j][0]) : 0u);
      const float v = H != 0 ? ord_val(H) : -FLT_MAX;
      const int k = H != 0 ? static_cast<int>(~Lo) : 0x7fffffff;
      if (q == 0 && H != 0) M[j] = fmaxf(M[j], v);
      if (lane == 0 && live[j]) {
        rr.tl[r0 + rs * j][q] = v;
        rr.tk[r0 + rs * j][q] = k;
      }
      if (H != 0 && t[j][0] == ((static_cast<uint64_t>(H) << 32) | Lo)) {
#pragma unroll
        for (int z = 0; z < BCAP - 1; ++z) t[j][z] = t[j][z + 1];
        t[j][BCAP - 1] = 0;
      }
    }
  }
  if constexpr (LSE) {
    double lse[NR];
    lse_exact<NR>(L, M, V, lse_scratch(HL, Vp), etab, lse);
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      if (lane == 0 && live[j]) {
        rr.lse[r0 + rs * j] = lse[j];
        rr.l0[r0 + rs * j] = L[j][0];
      }
    }
  }
}

// D for the whole CTA with the weight stages as scratch (WPipe::defer).
// (The arithmetic of decode_common.cuh's lse_cta_exps / lse_cta_chain, kept
// written out here: composed from those helpers ptxas allocates the beam
// kernel's frame loop differently and its GEMM phase runs ~3% slower.)
//  (a) row maxima (model.hpp:117-118), one warp per row;
//  (b) every exp(double(l_k) - max) of every row into E (row stride S, odd
//      so the chain lanes below hit distinct banks), one column per thread
//      -- all of the exp work spread over the 512 threads;
//  (c) warp 0 runs the reference's sequential sums (model.hpp:119-121), one
//      lane per row, while warps 1-15 pick the top-`beam` tokens.
// The index-order fp64 chain is ~V dependent DADDs per row; here it costs
// one warp V instructions for all rows, overlapped with the top-k.
template <int BCAP>
__device__ __forceinline__ void beam_reduce_cta(float* HL, double* E, int ecap, int Vp, int V, int beam, int R,
                                                RowRes rr, const uint64_t* etab, float* row_m) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < R; r += kWarps) {
    const float* L = HL + static_cast<int64_t>(r) * Vp;
    float mx = -FLT_MAX;
    for (int k = lane; k < V; k += 32) mx = fmaxf(mx, L[k]);
    mx = warp_max_f(mx);
    if (lane == 0) row_m[r] = mx;
  }
  __syncthreads();
  // Rows are zero-padded to V8 = V rounded up to 8 (+ 0.0 is exact once the
  // sum holds exp(0) = 1), so the chain below runs in whole groups of 8.
  constexpr int G8 = 8;
  const int V8 = (V + G8 - 1) / G8 * G8;
  int S = V8 + 1;
  if (S * R > ecap) S = V8;
  const int k = threadIdx.x;  // V8 <= kDecodeThreads
  auto arg = [&](int r) {
    return k < V ? rnntg_f64::xsub(static_cast<double>(HL[static_cast<int64_t>(r) * Vp + k]),
                                   static_cast<double>(row_m[r]))
                 : -1.0;
  };
  for (int r = 0; r < R; r += 2) {  // two rows per trip: independent exp chains interleave
    const int r1 = r + 1 < R ? r + 1 : r;
    const double x0 = arg(r), x1 = arg(r1);
    double y0 = exp_main(x0, etab), y1 = exp_main(x1, etab);
    if (__any_sync(0xffffffffu, exp_big(x0) || exp_big(x1))) {
      if (exp_big(x0)) y0 = rnntg_f64::exp_t(x0, etab);
      if (exp_big(x1)) y1 = rnntg_f64::exp_t(x1, etab);
    }
    if (k < V8) {
      E[r * S + k] = k < V ? y0 : 0.0;
      E[r1 * S + k] = k < V ? y1 : 0.0;
    }
  }
  __syncthreads();
  if (warp == 0) {
    if (lane < R) {
      // Software-pipelined: group q + 1's loads are in flight while group
      // q's 8 dependent DADDs run.
      const double* e = E + lane * S;
      double acc = 0.0, cur[G8], nxt[G8];
#pragma unroll
      for (int u = 0; u < G8; ++u) cur[u] = e[u];
      for (int q = G8; q < V8; q += G8) {
#pragma unroll
        for (int u = 0; u < G8; ++u) nxt[u] = e[q + u];
#pragma unroll
        for (int u = 0; u < G8; ++u) acc = rnntg_f64::xadd(acc, cur[u]);
#pragma unroll
        for (int u = 0; u < G8; ++u) cur[u] = nxt[u];
      }
#pragma unroll
      for (int u = 0; u < G8; ++u) acc = rnntg_f64::xadd(acc, cur[u]);
      rr.lse[lane] = rnntg_f64::xadd(static_cast<double>(row_m[lane]), rnntg_f64::log(acc));
      rr.l0[lane] = HL[static_cast<int64_t>(lane) * Vp];
    }
  } else {
    constexpr int kTw = kWarps - 1;  // top-k warps
    const int w = warp - 1;
    if (R <= kTw) {
      if (w < R) beam_row_reduce_n<BCAP, 1, false>(HL, Vp, V, beam, w, R, rr, etab);
    } else {
      beam_row_reduce_n<BCAP, 2, false>(HL, Vp, V, beam, w, R, rr, etab, kTw);
      if (w + 2 * kTw < R) beam_row_reduce_n<BCAP, 1, false>(HL, Vp, V, beam, w + 2 * kTw, R, rr, etab);
    }
  }
  __syncthreads();
}
template <int BCAP>
__device__ __noinline__ void beam_reduce_cta_ni(float* HL, double* E, int ecap, int Vp, int V, int beam, int R,
                                                RowRes rr, const uint64_t* etab, float* row_m) {
  beam_reduce_cta<BCAP>(HL, E, ecap, Vp, V, beam, R, rr, etab, row_m);
}

// Out-of-line copy for the time-sliced kernel instantiation (measured faster
// there than inlined; the single-launch kernel inlines it).
template <int BCAP, int NR>
__device__ __noinline__ void beam_row_reduce_ni(float* HL, int Vp, int V, int beam, int r0, int R,
                                                RowRes rr, const uint64_t* etab) {
  beam_row_reduce_n<BCAP, NR>(HL, Vp, V, beam, r0, R, rr, etab);
}

// E. one stream's frame (one warp).  Reference order (search.hpp:223-259 at
// S = 1): the extensions are cut to the beam first (prune_to_beam of
// next_level), then merged with the blank continuations by full-sequence
// equality, then the frame set is cut.  At the stream's last frame the
// winner (search.hpp:261-276) is traced back through the lattice.
template <int BCAP>
__device__ void beam_stream_step(const ModelView& m, Hyps& h, BeamCand* cand, uint32_t* bp, int t,
                                 int T, int fs, int beam, int merge_log, int length_norm,
                                 int max_total, RowRes rr, int32_t* tokens, int32_t* out_len,
                                 double* out_score, unsigned long long* ties) {
  const int lane = threadIdx.x & 31;
  BeamCand* merged = cand + BCAP * BCAP;  // [2 * BCAP]
  const int nh = h.nh;
  // Stage 1: every hypothesis' top-`beam` extensions; the global top `beam`
  // of those is the reference's pruned next_level.
  const int next = nh * beam;
  for (int c = lane; c < next; c += 32) {
    const int j = c / beam, q = c % beam;
    const int r = h.row[j];
    const bool may_emit = max_total <= 0 || h.len[j] < max_total;
    const int k = rr.tk[r][q];
    BeamCand& e = cand[c];
    e.score = (may_emit && k < m.V) ? h.score[j] + (static_cast<double>(rr.tl[r][q]) - rr.lse[r])
                                    : -INFINITY;
    e.parent = j;
    e.tok = k;
    e.len = h.len[j] + 1;
  }
  __syncwarp();
  int rank[2] = {0x7fffffff, 0x7fffffff};
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int c = lane + u * 32;
    if (c >= next || cand[c].score == -INFINITY) continue;
    const BeamCand a = cand[c];
    int rk = 0;
    for (int d = 0; d < next; ++d) {
      const BeamCand& b = cand[d];
      if (d == c || b.score == -INFINITY) continue;
      if (cand_before(b, b.score, a, a.score, bp, t, ties)) ++rk;
    }
    rank[u] = rk;
  }
  BeamCand sel[2];
#pragma unroll
  for (int u = 0; u < 2; ++u)
    if (rank[u] < beam) sel[u] = cand[lane + u * 32];
  int nsel = (rank[0] < beam ? 1 : 0) + (rank[1] < beam ? 1 : 0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nsel += __shfl_xor_sync(0xffffffffu, nsel, o);
  __syncwarp();
  // Stage 2 inputs: blank continuations in merged[0..nh), selected
  // extensions (with their new identities) in cand[0..nsel) by rank.
  if (lane < nh) {
    const int r = h.row[lane];
    BeamCand& b = merged[lane];
    b.score = h.score[lane] + (static_cast<double>(rr.l0[r]) - rr.lse[r]);
    b.h1 = h.h1[lane];
    b.h2 = h.h2[lane];
    b.p1 = h.p1[lane];
    b.p2 = h.p2[lane];
    b.parent = lane;
    b.tok = 0;
    b.len = h.len[lane];
    b.ctx = h.ctx[lane];
    b.last = h.last[lane];
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (rank[u] >= beam) continue;
    BeamCand e = sel[u];
    const int gp = e.parent;
    e.h1 = hash_ext1(h.h1[gp], e.tok);
    e.h2 = hash_ext2(h.h2[gp], e.tok);
    e.p1 = h.h1[gp];
    e.p2 = h.h2[gp];
    e.ctx = (h.ctx[gp] % m.V) * m.V + e.tok;
    e.last = e.tok;
    cand[rank[u]] = e;
  }
  __syncwarp();
  // merge_into (search.hpp:180-187): an extension ys_g+k equals the blank
  // continuation of hypothesis j iff |ys_j| = |ys_g|+1, last(ys_j) = k and
  // prefix(ys_j) = ys_g.
  // Each blank continuation j can equal at most one extension (extensions
  // are distinct sequences, and two extensions never merge with each other:
  // the reference compares them with the existing entries only), so lane q
  // merges extension q on its own; misses are appended in q order.
  int nm = nh;
  {
    int hit = -1;
    BeamCand e;
    if (lane < nsel) {
      e = cand[lane];
      for (int j = 0; j < nh; ++j)
        if (merged[j].last == e.tok && merged[j].len == e.len && merged[j].p1 == e.p1 &&
            merged[j].p2 == e.p2) {
          hit = j;
          break;
        }
    }
    const unsigned miss = __ballot_sync(0xffffffffu, lane < nsel && hit < 0);
    if (lane < nsel) {
      if (hit >= 0) {
        double& sc = merged[hit].score;
        if (merge_log) {  // log_add, common.hpp:48-54 (glibc exp / log1p bits)
          sc = rnntg_f64::log_add(sc, e.score);
        } else {
          sc = sc > e.score ? sc : e.score;
        }
      } else {
        merged[nh + __popc(miss & ((1u << lane) - 1u))] = e;
      }
    }
    nm = nh + __popc(miss);
  }
  __syncwarp();
  // prune_to_beam of the frame set by hyp_better.
  int myrank = 0x7fffffff;
  BeamCand mine;
  if (lane < nm) {
    mine = merged[lane];
    int rk = 0;
    for (int d = 0; d < nm; ++d) {
      if (d == lane) continue;
      if (cand_before(merged[d], merged[d].score, mine, mine.score, bp, t, ties)) ++rk;
    }
    myrank = rk;
  }
  __syncwarp();
  if (myrank < beam) {
    h.score[myrank] = mine.score;
    h.h1[myrank] = mine.h1;
    h.h2[myrank] = mine.h2;
    h.p1[myrank] = mine.p1;
    h.p2[myrank] = mine.p2;
    h.ctx[myrank] = mine.ctx;
    h.len[myrank] = mine.len;
    h.last[myrank] = mine.last;
    bp[(t + 1) * kMaxBeam + myrank] =
        (static_cast<uint32_t>(mine.tok) << 8) | static_cast<uint32_t>(mine.parent);
  }
  if (lane == 0) h.nh = min(nm, beam);
  __syncwarp();
  if (t + 1 == T && lane == 0) {
    const int nf = h.nh;
    int best = 0;
    for (int j = 1; j < nf; ++j) {
      const double kj = length_norm ? h.score[j] / max(1, h.len[j]) : h.score[j];
      const double kb = length_norm ? h.score[best] / max(1, h.len[best]) : h.score[best];
      BeamCand a, b;
      a.len = h.len[j];
      a.parent = j;
      a.tok = 0;
      b.len = h.len[best];
      b.parent = best;
      b.tok = 0;
      if (cand_before(a, kj, b, kb, bp, T, ties)) best = j;
    }
    *out_score = h.score[best];
    *out_len = h.len[best];
    int pos = h.len[best];
    int tau = T, slot = best;
    while (tau > 0) {
      const uint32_t e = bp[tau * kMaxBeam + slot];
      --tau;
      slot = static_cast<int>(e & 0xffu);
      const int tok = static_cast<int>(e >> 8);
      if (tok != 0) tokens[fs + --pos] = tok;
    }
  }
}

// Out-of-line call for the time-sliced instantiation (RNNTG_SL_STEP_NI).
template <int BCAP>
__device__ __noinline__ void beam_stream_step_ni(const ModelView& m, Hyps& h, BeamCand* cand, uint32_t* bp, int t,
                                                 int T, int fs, int beam, int merge_log, int length_norm,
                                                 int max_total, RowRes rr, int32_t* tokens, int32_t* out_len,
                                                 double* out_score, unsigned long long* ties) {
  beam_stream_step<BCAP>(m, h, cand, bp, t, T, fs, beam, merge_log, length_norm, max_total, rr, tokens, out_len,
                         out_score, ties);
}

// Development knob: GEMM over this many rows every frame (0 = off;
// RNNTG_DBG_FORCE_R, the joiner GEMM's marginal-rate experiment).
struct DbgKnobs {
  int32_t dbg_force_r;
};

// SL: time-sliced launch (frames [sl.t0, sl.t1), hypothesis sets resumed
// from / kept in sl.state).  A separate instantiation so the single-launch
// kernel's code is untouched by the slice plumbing (ptxas's register
// allocation of the frame loop is sensitive to it: ~1-2%).
template <int BCAP, bool TC, bool SL = false>
__global__ void __launch_bounds__(kDecodeThreads, 1)
    beam_kernel(ModelView m, const float* __restrict__ pe,
                const int32_t* __restrict__ frame_splits, int32_t B, int32_t G,
                int32_t beam, int32_t merge_log, int32_t length_norm,
                int32_t max_total, uint32_t* __restrict__ backptr,
                int32_t* __restrict__ tokens, int32_t* __restrict__ lengths,
                double* __restrict__ scores,
                unsigned long long* __restrict__ counters, DbgKnobs fp, BeamSlice sl) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* HL = reinterpret_cast<float*>(smem_raw);
  const int hl_floats = hl_floats_of(m.J, m.Vp);
  // weight stages: two kBK-row fp32 chunks, or (bf16 variant) kTcStages
  // 16 KB bf16 chunks = the area of two 16-row fp32 chunks
  const int wst = TC ? 16 * m.Vp : kBK * m.Vp;
  float* W0 = HL + hl_floats;
  float* W1 = W0 + wst;
  BeamSmem& S = *reinterpret_cast<BeamSmem*>(W1 + wst);
  Hyps* H = reinterpret_cast<Hyps*>(&S + 1);          // [G]
  BeamCand* C = reinterpret_cast<BeamCand*>(H + G);   // [G][BCAP*BCAP + 2*BCAP]
  constexpr int kCandPerStream = BCAP * BCAP + 2 * BCAP;
  // bf16 variant: tensor-core operand tile and its barriers after the rest.
  unsigned char* hb = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(C + G * kCandPerStream) + 1023) & ~static_cast<uintptr_t>(1023));
  TcBars* tb = reinterpret_cast<TcBars*>(hb + kRowCap * m.J * 2);

  const int s0 = blockIdx.x * G;
  const int ns = min(G, B - s0);
  if (ns <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // The pipe descriptor lives in shared memory: its fields are read where a
  // chunk is waited for or issued instead of pinning ~14 registers across
  // every phase (register pressure here costs the GEMM its LDS prefetch).
  const WPipe& pipe = S.pipe;
  if (threadIdx.x == 0) {
    S.pipe = make_wpipe(W0, W1, S.bar, S.wcur, m);
    // exact fp32 joiner: the row reduction borrows both weight stages
    S.pipe.defer = (!TC && S.pipe.nc >= 2 && m.Vp <= kDecodeThreads) ? 1 : 0;
  }
  TcPipe tp{smem_u32(W0), tb->full, tb->empty, &tb->done, smem_u32(hb), 0u, m.J / kTcBK};

  int32_t tmax = 0;
  for (int i = 0; i < ns; ++i)
    tmax = max(tmax, frame_splits[s0 + i + 1] - frame_splits[s0 + i]);
  // Only t_end stays live across the frame loop (it replaces tmax); sl.* are
  // kernel parameters (constant bank), re-read where needed.
  const int32_t t_end = SL ? min(sl.t1, tmax) : tmax;
  if (SL && sl.t0 > 0) {  // resume: this CTA's hypothesis sets
    copy_hyps(H, sl.state + s0, ns);
  } else {
    for (int i = threadIdx.x; i < ns; i += kDecodeThreads) {
      Hyps& h = H[i];
      h.nh = 1;
      h.score[0] = 0.0;
      h.ctx[0] = 0;
      h.len[0] = 0;
      h.last[0] = -1;
      h.h1[0] = 0x243f6a8885a308d3ull;
      h.h2[0] = 0x13198a2e03707344ull;
      h.p1[0] = h.p2[0] = 0;
    }
  }
  if (threadIdx.x < 16) S.stat[threadIdx.x] = 0;
  load_exp_table(S.etab);
  if (threadIdx.x == 0) {
    if constexpr (TC) {
      for (int i = 0; i < kTcStages; ++i) {
        mbar_init(&tb->full[i], 1);
        mbar_init(&tb->empty[i], 1);
      }
      mbar_init(&tb->done, 1);
    } else {
      mbar_init(&S.bar[0], 1);
      mbar_init(&S.bar[1], 1);
    }
    fence_mbar_init();
  }
  if constexpr (TC) {
    if (warp == 0) tc::tmem_alloc(&tb->tmem_addr, kTmemCols);
    tc::fence_before_sync();
  }
  __syncthreads();
  if constexpr (TC) {
    tc::fence_after_sync();
    tp.tmem = tb->tmem_addr;
    if (threadIdx.x == 0)
      for (int i = 0; i < kTcStages; ++i) tc_issue(tp, m, i);
  } else if (threadIdx.x == 0) {
    wpipe_issue(pipe, m, 0);
    wpipe_issue(pipe, m, 1);
  }
  uint32_t g = 0;
  // Per-CTA counters live in shared memory (thread 0 accumulates; ties by
  // shared atomics) so no register is held across the GEMM for them.
  unsigned long long* st = S.stat;
  long long* pst = reinterpret_cast<long long*>(S.stat);

  // One block of frames [t_begin, t_end) (the block structure is kept: the
  // frame loop's register allocation is sensitive to its shape).
  const int32_t t_begin = SL ? sl.t0 : 0;
  const int32_t TB = max(1, t_end - t_begin);
  for (int32_t tb = t_begin; tb < t_end; tb += TB) {
  const int32_t te = min(tb + TB, t_end);
  for (int32_t t = tb; t < te; ++t) {
    // A. rows: distinct contexts per live stream (lane = stream, G <= 32).
    if (warp == 0) {
      const int R0 = beam_rows(H, ns, frame_splits + s0, t, S.row_pe, S.row_ctx);
      if (lane == 0) S.nrows = R0;
    }
    __syncthreads();
    const int R = S.nrows;
    if (threadIdx.x == 0) {
      st[1] += R;
      st[5] += (m.Vp == 512 && R > 4 && R < 28) ? R : ((R + 3) & ~3);
    }
    long long c0 = clock64();
    if constexpr (TC)
      build_h_tc(m, pe, S.row_pe, S.row_ctx, R, R <= 16 ? 16 : 32, hb);
    else
      build_h(m, pe, S.row_pe, S.row_ctx, R, HL, pst + 2);
    long long c1 = clock64();
    if (threadIdx.x == 0) pst[6] += pst[2] - c0;
    // Next frame's encoder projections into L2 while the GEMM runs (each
    // stream's pe row is 2 KB of HBM read once; the h build then hits L2).
    {
      const int lines = (m.J * 4 + 127) >> 7;
      for (int x = threadIdx.x; x < ns * lines; x += kDecodeThreads) {
        const int i = x / lines, l = x - i * lines;
        const int32_t f = frame_splits[s0 + i];
        if (t + 1 < frame_splits[s0 + i + 1] - f)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pe + static_cast<int64_t>(f + t + 1) * m.J + l * 32));
      }
    }
    if constexpr (TC)
      tc_gemm(m, tp, g, static_cast<uint32_t>(t), HL, R);
    else
      joiner_gemm(m, pipe, g, HL, fp.dbg_force_r > 0 ? fp.dbg_force_r : R, pst + 7);
    long long c2 = clock64();

    // D. per row: lse, blank logit, top-`beam` tokens k >= 1 by (logit desc,
    // token asc).  Each lane keeps a sorted local top-kMaxBeam, then `beam`
    // warp-wide pops.
    const RowRes rr{S.row_lse, S.row_l0, S.row_tl, S.row_tk};
    if (!TC && pipe.defer) {
      if constexpr ((SL && RNNTG_SL_RR_NI) || (!SL && RNNTG_MAIN_RR_NI))
        beam_reduce_cta_ni<BCAP>(HL, reinterpret_cast<double*>(W0), wst, m.Vp, m.V, beam, R, rr, S.etab, S.row_m);
      else
        beam_reduce_cta<BCAP>(HL, reinterpret_cast<double*>(W0), wst, m.Vp, m.V, beam, R, rr, S.etab, S.row_m);
      wpipe_issue_next(pipe, m, g);
    } else if constexpr ((SL && RNNTG_SL_RR_NI) || (!SL && RNNTG_MAIN_RR_NI)) {
      if (R <= kWarps) {
        if (warp < R) beam_row_reduce_ni<BCAP, 1>(HL, m.Vp, m.V, beam, warp, R, rr, S.etab);
      } else if (warp < R - kWarps || warp < kWarps) {
        beam_row_reduce_ni<BCAP, 2>(HL, m.Vp, m.V, beam, warp, R, rr, S.etab);
      }
    } else {
      if (R <= kWarps) {
        if (warp < R) beam_row_reduce_n<BCAP, 1>(HL, m.Vp, m.V, beam, warp, R, rr, S.etab);
      } else if (warp < R - kWarps || warp < kWarps) {
        beam_row_reduce_n<BCAP, 2>(HL, m.Vp, m.V, beam, warp, R, rr, S.etab);
      }
    }
    __syncthreads();

    long long c3 = clock64();
    // E. beam step, one warp per stream.  Reference order (search.hpp:
    // 223-259 at S = 1): the extensions are cut to the beam first
    // (prune_to_beam of next_level), then merged with the blank
    // continuations by full-sequence equality, then the frame set is cut.
    for (int i = warp; i < ns; i += kWarps) {
      const int32_t fs = frame_splits[s0 + i];
      const int32_t T = frame_splits[s0 + i + 1] - fs;
      if (t >= T) continue;
      if constexpr ((SL && RNNTG_SL_STEP_NI) || (!SL && RNNTG_MAIN_STEP_NI))
        beam_stream_step_ni<BCAP>(m, H[i], C + static_cast<int64_t>(i) * kCandPerStream,
                                  backptr + static_cast<int64_t>(fs + s0 + i) * kMaxBeam, t, T, fs, beam,
                                  merge_log, length_norm, max_total, rr, tokens, lengths + s0 + i,
                                  scores + s0 + i, &st[4]);
      else
        beam_stream_step<BCAP>(m, H[i], C + static_cast<int64_t>(i) * kCandPerStream,
                               backptr + static_cast<int64_t>(fs + s0 + i) * kMaxBeam, t, T, fs, beam,
                               merge_log, length_norm, max_total, rr, tokens, lengths + s0 + i,
                               scores + s0 + i, &st[4]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long c4 = clock64();
      pst[8] += c1 - c0;
      pst[9] += c2 - c1;
      pst[10] += c3 - c2;
      pst[11] += c4 - c3;
    }
  }
  }
  // Zero-frame streams: empty result, score 0.
  for (int i = threadIdx.x; i < ns; i += kDecodeThreads)
    if (frame_splits[s0 + i + 1] == frame_splits[s0 + i]) {
      lengths[s0 + i] = 0;
      scores[s0 + i] = 0.0;
    }
  if (SL)  // sliced launch: keep the hypothesis sets for the next slice
    copy_hyps(sl.state + s0, H, ns);
  __syncthreads();
  if (threadIdx.x < 16 && threadIdx.x != 0 && threadIdx.x != 2 && st[threadIdx.x] != 0)
    atomicAdd(&counters[threadIdx.x], st[threadIdx.x]);
  if constexpr (TC) {
    // Chunks g .. g+kTcStages-2 were prefetched for a frame that never came.
    if (threadIdx.x == 0)
      for (uint32_t x = g; x < g + kTcStages - 1; ++x) mbar_wait(&tb->full[x % kTcStages], (x / kTcStages) & 1u);
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
      tc::fence_after_sync();
      tc::tmem_dealloc(tp.tmem, kTmemCols);
    }
  }
  if (threadIdx.x == 0) {
    if constexpr (!TC) {
      mbar_wait(&S.bar[g & 1u], (g >> 1) & 1u);
      mbar_wait(&S.bar[(g + 1) & 1u], ((g + 1) >> 1) & 1u);
    }
    unsigned long long sf = 0;  // frames decoded by this launch
    for (int i = 0; i < ns; ++i)
      sf += SL ? max(0, min(frame_splits[s0 + i + 1] - frame_splits[s0 + i], t_end) - sl.t0)
               : frame_splits[s0 + i + 1] - frame_splits[s0 + i];
    atomicAdd(&counters[0], sf);
  }
}

// ---------------------------------------------------------------------------
// Modified beam search with S > 1 symbols per frame (beam_search,
// search.hpp:206-277, any max_symbols).  Per frame and stream: level := the
// beam; repeat { one joiner row per distinct context of the level; every
// level hypothesis' blank continuation is merged into next_frame (by full
// sequence identity, max or log_add); the level's extensions are cut to the
// beam and become the next level } until the level is empty or `cap`
// sub-steps ran (then the level is merged into next_frame with no score
// factor); next_frame is cut to the beam.  Each sub-step is one CTA-wide
// GEMM pass over the streams whose level is non-empty.  Sequences are kept
// as nodes (parent, token) in a per-stream HBM pool (only extensions create
// nodes; a blank continuation is its hypothesis' own node), which serves the
// traceback and hyp_better's lexicographic tie rule.
// ---------------------------------------------------------------------------
constexpr int kNfCap = kMaxBeam * 11;  // next_frame entries: beam x (cap + 1), cap <= 10

struct NfEntry {
  double score;
  uint64_t h1, h2;
  int32_t len, ctx, last, node;
};

struct MStream {
  int32_t node[kMaxBeam];  // level hypotheses' pool nodes
  NfEntry nf[kNfCap];
  int32_t nf_n;
  int32_t pool_n;
  BeamCand cand[kMaxBeam * kMaxBeam];
};

struct MultiSmem {
  uint64_t etab[256];  // glibc exp table (lse_exact)
  unsigned long long stat[16];
  uint64_t bar[2];
  uint32_t wcur[2];
  int64_t row_pe[kRowCap];
  int32_t row_ctx[kRowCap];
  double row_lse[kRowCap];
  float row_l0[kRowCap];
  float row_tl[kRowCap][kMaxBeam];
  int32_t row_tk[kRowCap][kMaxBeam];
  int32_t nrows;
};

// Lexicographic order of two equal-length sequences given as pool nodes
// (<0, 0, >0): walk back in lockstep, the last difference seen is the first
// position where they differ.
__device__ int node_lex(const int2* __restrict__ pool, int a, int b) {
  int res = 0;
  while (a != b) {
    const int2 x = pool[a], y = pool[b];
    if (x.y != y.y) res = x.y < y.y ? -1 : 1;
    a = x.x;
    b = y.x;
  }
  return res;
}

// hyp_better (search.hpp:172-178) for (key, len, node [, pending token]).
__device__ __forceinline__ bool seq_before(double ka, int la, int na, int ta, double kb, int lb, int nb,
                                           int tb, const int2* pool, unsigned long long* ties) {
  if (ka != kb) return ka > kb;
  if (la != lb) return la < lb;
  ++*ties;
  // equal lengths: compare the parents' sequences, then the pending tokens
  const int c = node_lex(pool, na, nb);
  if (c != 0) return c < 0;
  return ta < tb;
}

__device__ __forceinline__ void nf_merge(NfEntry& e, double v, int merge_log) {
  if (merge_log) {  // log_add, common.hpp:48-54 (glibc exp / log1p bits)
    e.score = rnntg_f64::log_add(e.score, v);
  } else {
    e.score = e.score > v ? e.score : v;
  }
}

// Merges level hypotheses j (lane j < nl) into next_frame with scores v_j.
// Level hypotheses are distinct sequences, so each lane's entry is hit by
// no other lane of this call; misses are appended in lane order.
__device__ __forceinline__ void nf_merge_level(MStream& st, const Hyps& lev, int nl, double v, int merge_log) {
  const int lane = threadIdx.x & 31;
  int hit = -1;
  const int n0 = st.nf_n;
  if (lane < nl) {
    for (int q = 0; q < n0; ++q) {
      const NfEntry& e = st.nf[q];
      if (e.len == lev.len[lane] && e.h1 == lev.h1[lane] && e.h2 == lev.h2[lane]) {
        hit = q;
        break;
      }
    }
  }
  const unsigned miss = __ballot_sync(0xffffffffu, lane < nl && hit < 0);
  if (lane < nl) {
    if (hit >= 0) {
      nf_merge(st.nf[hit], v, merge_log);
    } else {
      NfEntry& e = st.nf[n0 + __popc(miss & ((1u << lane) - 1u))];
      e.score = v;
      e.h1 = lev.h1[lane];
      e.h2 = lev.h2[lane];
      e.len = lev.len[lane];
      e.ctx = lev.ctx[lane];
      e.last = lev.last[lane];
      e.node = st.node[lane];
    }
  }
  __syncwarp();
  if (lane == 0) st.nf_n = n0 + __popc(miss);
  __syncwarp();
}

template <int BCAP>
__global__ void __launch_bounds__(kDecodeThreads, 1)
    beam_multi_kernel(ModelView m, const float* __restrict__ pe, const int32_t* __restrict__ frame_splits,
                      int32_t B, int32_t G, int32_t cap, int32_t count_capped, int32_t beam,
                      int32_t merge_log, int32_t length_norm, int32_t max_total, int2* __restrict__ pool,
                      int32_t* __restrict__ tokens, int32_t* __restrict__ lengths, double* __restrict__ scores,
                      unsigned long long* __restrict__ counters) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* HL = reinterpret_cast<float*>(smem_raw);
  const int hl_floats = hl_floats_of(m.J, m.Vp);
  float* W0 = HL + hl_floats;
  float* W1 = W0 + kBKSmall * m.Vp;
  MultiSmem& S = *reinterpret_cast<MultiSmem*>(W1 + kBKSmall * m.Vp);
  Hyps* L = reinterpret_cast<Hyps*>(&S + 1);         // [G] levels
  MStream* MS = reinterpret_cast<MStream*>(L + G);   // [G]
  const int s0 = blockIdx.x * G;
  const int ns = min(G, B - s0);
  if (ns <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const WPipe pipe = make_wpipe(W0, W1, S.bar, S.wcur, m, kBKSmall);

  int32_t tmax = 0;
  for (int i = 0; i < ns; ++i) tmax = max(tmax, frame_splits[s0 + i + 1] - frame_splits[s0 + i]);
  for (int i = threadIdx.x; i < ns; i += kDecodeThreads) {
    Hyps& h = L[i];  // the beam {[]: 0.0}
    h.nh = 1;
    h.score[0] = 0.0;
    h.ctx[0] = 0;
    h.len[0] = 0;
    h.last[0] = -1;
    h.h1[0] = 0x243f6a8885a308d3ull;
    h.h2[0] = 0x13198a2e03707344ull;
    h.p1[0] = h.p2[0] = 0;
    MS[i].node[0] = 0;
    MS[i].pool_n = 1;
    const int64_t pb = static_cast<int64_t>(frame_splits[s0 + i]) * cap * kMaxBeam + s0 + i;
    pool[pb] = make_int2(0, 0);  // root
  }
  if (threadIdx.x < 16) S.stat[threadIdx.x] = 0;
  load_exp_table(S.etab);
  if (threadIdx.x == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    wpipe_issue(pipe, m, 0);
    wpipe_issue(pipe, m, 1);
  }
  uint32_t g = 0;

  for (int32_t t = 0; t < tmax; ++t) {
    for (int i = warp; i < ns; i += kWarps)
      if (lane == 0) MS[i].nf_n = 0;
    for (int32_t n = 0;; ++n) {
      __syncthreads();
      if (n == cap) {  // emission budget exhausted: forced advance, blank prob 1
        for (int i = warp; i < ns; i += kWarps) {
          const int32_t T = frame_splits[s0 + i + 1] - frame_splits[s0 + i];
          if (t >= T || L[i].nh == 0) continue;
          // scores unchanged; merge each level hypothesis with its own score
          const double v = lane < L[i].nh ? L[i].score[lane] : 0.0;
          nf_merge_level(MS[i], L[i], L[i].nh, v, merge_log);
          if (count_capped && lane == 0) atomicAdd(&S.stat[13], 1ull);
        }
        break;
      }
      if (warp == 0) {
        const int R0 = beam_rows(L, ns, frame_splits + s0, t, S.row_pe, S.row_ctx);
        if (lane == 0) S.nrows = R0;
      }
      __syncthreads();
      const int R = S.nrows;
      if (R == 0) break;  // every live level is empty
      if (threadIdx.x == 0) S.stat[1] += R;
      build_h(m, pe, S.row_pe, S.row_ctx, R, HL);
      joiner_gemm(m, pipe, g, HL, R);
      const RowRes rr{S.row_lse, S.row_l0, S.row_tl, S.row_tk};
      if (R <= kWarps) {
        if (warp < R) beam_row_reduce_n<BCAP, 1>(HL, m.Vp, m.V, beam, warp, R, rr, S.etab);
      } else if (warp < R - kWarps || warp < kWarps) {
        beam_row_reduce_n<BCAP, 2>(HL, m.Vp, m.V, beam, warp, R, rr, S.etab);
      }
      __syncthreads();
      for (int i = warp; i < ns; i += kWarps) {
        const int32_t fs = frame_splits[s0 + i];
        const int32_t T = frame_splits[s0 + i + 1] - fs;
        Hyps& h = L[i];
        MStream& st = MS[i];
        const int nl = h.nh;
        if (t >= T || nl == 0) continue;
        const int64_t pb = static_cast<int64_t>(fs) * cap * kMaxBeam + s0 + i;
        const int2* P = pool + pb;
        // blank continuations into next_frame: score + lp[0]
        const double vb = lane < nl ? h.score[lane] + (static_cast<double>(rr.l0[h.row[lane]]) - rr.lse[h.row[lane]]) : 0.0;
        nf_merge_level(st, h, nl, vb, merge_log);
        // extensions: each hypothesis' top-`beam` tokens, then the level's top `beam`
        BeamCand* cand = st.cand;
        const int next = nl * beam;
        for (int c = lane; c < next; c += 32) {
          const int j = c / beam, q = c % beam;
          const int r = h.row[j];
          const bool may_emit = max_total <= 0 || h.len[j] < max_total;
          const int k = rr.tk[r][q];
          BeamCand& e = cand[c];
          e.score = (may_emit && k < m.V) ? h.score[j] + (static_cast<double>(rr.tl[r][q]) - rr.lse[r]) : -INFINITY;
          e.parent = j;
          e.tok = k;
          e.len = h.len[j] + 1;
        }
        __syncwarp();
        int rank[2] = {0x7fffffff, 0x7fffffff};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = lane + u * 32;
          if (c >= next || cand[c].score == -INFINITY) continue;
          const BeamCand a = cand[c];
          int rk = 0;
          for (int d = 0; d < next; ++d) {
            const BeamCand& b = cand[d];
            if (d == c || b.score == -INFINITY) continue;
            if (seq_before(b.score, b.len, st.node[b.parent], b.tok, a.score, a.len, st.node[a.parent], a.tok, P,
                           &S.stat[4]))
              ++rk;
          }
          rank[u] = rk;
        }
        BeamCand sel[2];
        int selnode[2] = {0, 0};
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (rank[u] < beam) sel[u] = cand[lane + u * 32];
        int nsel = (rank[0] < beam ? 1 : 0) + (rank[1] < beam ? 1 : 0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nsel += __shfl_xor_sync(0xffffffffu, nsel, o);
        // new level (slot = rank) with fresh pool nodes (parent, token)
        const int pn = st.pool_n;
        uint64_t h1n[2], h2n[2];
        int ctxn[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (rank[u] >= beam) continue;
          const int gp = sel[u].parent;
          h1n[u] = hash_ext1(h.h1[gp], sel[u].tok);
          h2n[u] = hash_ext2(h.h2[gp], sel[u].tok);
          ctxn[u] = (h.ctx[gp] % m.V) * m.V + sel[u].tok;
          selnode[u] = pn + rank[u];
          pool[pb + selnode[u]] = make_int2(st.node[gp], sel[u].tok);
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (rank[u] >= beam) continue;
          const int rk = rank[u];
          h.score[rk] = sel[u].score;
          h.h1[rk] = h1n[u];
          h.h2[rk] = h2n[u];
          h.ctx[rk] = ctxn[u];
          h.len[rk] = sel[u].len;
          h.last[rk] = sel[u].tok;
          st.node[rk] = selnode[u];
        }
        __syncwarp();
        if (lane == 0) {
          h.nh = min(nsel, beam);
          st.pool_n = pn + min(nsel, beam);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // next_frame cut to the beam (prune_to_beam): rank every entry by hyp_better
    for (int i = warp; i < ns; i += kWarps) {
      const int32_t fs = frame_splits[s0 + i];
      const int32_t T = frame_splits[s0 + i + 1] - fs;
      if (t >= T) continue;
      Hyps& h = L[i];
      MStream& st = MS[i];
      const int64_t pb = static_cast<int64_t>(fs) * cap * kMaxBeam + s0 + i;
      const int2* P = pool + pb;
      const int nn = st.nf_n;
      int rk3[3] = {0x7fffffff, 0x7fffffff, 0x7fffffff};
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int c = lane + 32 * u;
        if (c >= nn) continue;
        const NfEntry& a = st.nf[c];
        int rk = 0;
        for (int d = 0; d < nn; ++d) {
          if (d == c) continue;
          const NfEntry& b = st.nf[d];
          if (seq_before(b.score, b.len, b.node, -1, a.score, a.len, a.node, -1, P, &S.stat[4])) ++rk;
        }
        rk3[u] = rk;
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        if (rk3[u] >= beam) continue;
        const NfEntry& a = st.nf[lane + 32 * u];
        const int rk = rk3[u];
        h.score[rk] = a.score;
        h.h1[rk] = a.h1;
        h.h2[rk] = a.h2;
        h.ctx[rk] = a.ctx;
        h.len[rk] = a.len;
        h.last[rk] = a.last;
        st.node[rk] = a.node;
      }
      __syncwarp();
      if (lane == 0) h.nh = min(nn, beam);
      __syncwarp();
      if (t + 1 == T && lane == 0) {  // final answer (search.hpp:261-276)
        int best = 0;
        for (int j = 1; j < h.nh; ++j) {
          const double kj = length_norm ? h.score[j] / max(1, h.len[j]) : h.score[j];
          const double kb = length_norm ? h.score[best] / max(1, h.len[best]) : h.score[best];
          if (seq_before(kj, h.len[j], st.node[j], -1, kb, h.len[best], st.node[best], -1, P, &S.stat[4]))
            best = j;
        }
        scores[s0 + i] = h.score[best];
        lengths[s0 + i] = h.len[best];
        int pos = h.len[best];
        int nd = st.node[best];
        const int64_t ob = static_cast<int64_t>(cap) * fs;
        while (nd != 0) {
          const int2 e = P[nd];
          tokens[ob + --pos] = e.y;
          nd = e.x;
        }
      }
    }
  }
  for (int i = threadIdx.x; i < ns; i += kDecodeThreads)
    if (frame_splits[s0 + i + 1] == frame_splits[s0 + i]) {
      lengths[s0 + i] = 0;
      scores[s0 + i] = 0.0;
    }
  __syncthreads();
  if (threadIdx.x < 16 && threadIdx.x != 0 && S.stat[threadIdx.x] != 0)
    atomicAdd(&counters[threadIdx.x], S.stat[threadIdx.x]);
  if (threadIdx.x == 0) {
    mbar_wait(&S.bar[g & 1u], (g >> 1) & 1u);
    mbar_wait(&S.bar[(g + 1) & 1u], ((g + 1) >> 1) & 1u);
    unsigned long long sf = 0;
    for (int i = 0; i < ns; ++i) sf += frame_splits[s0 + i + 1] - frame_splits[s0 + i];
    atomicAdd(&counters[0], sf);
  }
}

template <int BCAP>
cudaError_t launch_beam_multi(const DecodeArgs& a, cudaStream_t s) {
  const ModelView m = view_of(*a.m);
  const int G = a.streams_per_cta;
  const size_t smem = smem_common(m, kBKSmall) + sizeof(MultiSmem) + (sizeof(Hyps) + sizeof(MStream)) * G;
  cudaError_t e = cudaFuncSetAttribute(beam_multi_kernel<BCAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int grid = (a.B + G - 1) / G;
  beam_multi_kernel<BCAP><<<grid, kDecodeThreads, smem, s>>>(
      m, a.pe, a.frame_splits, a.B, G, a.symbol_cap, a.count_capped, a.beam_size, a.merge_op, a.length_norm,
      a.max_total, static_cast<int2*>(a.node_pool), a.tokens, a.lengths, a.scores, a.counters);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Small-batch modified beam search on thread-block clusters (beam_search at
// S = 1, search.hpp:206-277).  With fewer streams than a
// few per SM the persistent kernel is latency bound: each SM streams all of
// out_w (1 MB) from L2 per frame for ~4 joiner rows and pays the fixed
// per-frame phases (h build, exact normaliser chain, beam step) for one or
// two streams.  Here a cluster of kBc = 8 CTAs serves G <= 64 / beam
// streams:
//  - CTA c keeps out_w columns [64c, 64c+64) resident in shared memory for
//    the whole utterance (no weight traffic after the first frame);
//  - the cluster builds the h rows of its joiner rows (<= 64, in passes of
//    32) together: CTA c evaluates k in [cJ/8, (c+1)J/8) of every row and
//    stores the slice into every CTA (16-byte st.async completing an
//    mbarrier transaction, no cluster barrier);
//  - every CTA computes its column slice of the logits (thread = column x
//    up to 4 rows, k-contiguous LDS.128 operands, sequential FMUL/FADD in
//    k, the reference's order); row r's slices go to CTA (r mod 8) by
//    st.async, which reduces it: exact normaliser (lse_cta_exps /
//    lse_cta_chain) with the top-`beam` tokens picked meanwhile, results
//    pushed to CTA 0;
//  - CTA 0 runs the beam steps (warp per stream: the persistent kernel's
//    beam_stream_step) and the next frame's rows; the others read the row
//    table back through DSMEM.
// Two cluster barriers per frame (three with a second pass).  Same
// arithmetic as the persistent kernel (identical tokens, bit-equal scores).
// ---------------------------------------------------------------------------
constexpr int kBc = 8;            // CTAs per cluster (portable maximum)
constexpr int kBcCols = 64;       // out_w columns per CTA (Vp = 512)
constexpr int kBcRows = 64;       // joiner rows per cluster frame
constexpr int kBcPass = 32;       // rows per h / GEMM pass
constexpr int kBcLocal = kBcRows / kBc;  // rows reduced per CTA

struct BcSmem {
  uint64_t hbar;  // this pass's h slices from every CTA have landed
  uint64_t lbar;  // this frame's logit slices of the rows reduced here have landed
  uint64_t etab[256];
  unsigned long long stat[8];
  int32_t R;
  int64_t row_pe[kBcRows];
  int32_t row_ctx[kBcRows];
  // CTA 0: every row's reduction results (the beam steps' RowRes)
  double row_lse[kBcRows];
  float row_l0[kBcRows];
  float row_tl[kBcRows][kMaxBeam];
  int32_t row_tk[kBcRows][kMaxBeam];
  // the rows this CTA reduces (local index r / kBc)
  double loc_lse[kBcLocal];
  float loc_l0[kBcLocal];
  float loc_tl[kBcLocal][kMaxBeam];
  int32_t loc_tk[kBcLocal][kMaxBeam];
  float loc_m[kBcLocal];
};

template <int BCAP>
__global__ void __launch_bounds__(kDecodeThreads, 1)
    beam_cluster_kernel(ModelView m, const float* __restrict__ pe, const int32_t* __restrict__ frame_splits,
                        int32_t B, int32_t G, int32_t beam, int32_t merge_log, int32_t length_norm,
                        int32_t max_total, uint32_t* __restrict__ backptr, int32_t* __restrict__ tokens,
                        int32_t* __restrict__ lengths, double* __restrict__ scores,
                        unsigned long long* __restrict__ counters) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int cl = blockIdx.x / kBc;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int JS = m.J + 4;     // k-contiguous rows, +4 floats: 16-byte column reads spread over the banks
  const int Sl = m.J / kBc;   // this CTA's k-slice of every h row
  float* Ws = reinterpret_cast<float*>(smem_raw);      // [64][J+4] out_w column slice, column-major
  float* Hs = Ws + kBcCols * JS;                       // [32][J+4] h rows of a pass (scratch after the GEMM)
  float* recv = Hs + kBcPass * JS;                     // [kBcLocal][Vp] logits of the rows reduced here
  BcSmem& S = *reinterpret_cast<BcSmem*>(recv + kBcLocal * m.Vp);
  Hyps* H = reinterpret_cast<Hyps*>(&S + 1);            // CTA 0: [G]
  BcSmem& S0 = *cluster.map_shared_rank(&S, 0);
  constexpr int kCandPerStream = BCAP * BCAP + 2 * BCAP;
  BeamCand* C = reinterpret_cast<BeamCand*>(Hs);       // CTA 0, during the beam steps

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s0 = cl * G;
  const int ns = max(0, min(G, B - s0));
  const int c0 = rank * kBcCols;
  for (int x = threadIdx.x; x < m.J * kBcCols; x += kDecodeThreads) {
    const int k = x / kBcCols, c = x - k * kBcCols;
    Ws[c * JS + k] = m.out_wt[static_cast<int64_t>(k) * m.Vp + c0 + c];
  }
  if (threadIdx.x == 0) {
    mbar_init(&S.hbar, 1);
    mbar_init(&S.lbar, 1);
    fence_mbar_init();
  }
  load_exp_table(S.etab);
  if (threadIdx.x < 8) S.stat[threadIdx.x] = 0;
  int32_t tmax = 0;
  for (int i = 0; i < ns; ++i) tmax = max(tmax, frame_splits[s0 + i + 1] - frame_splits[s0 + i]);
  if (rank == 0) {
    for (int i = threadIdx.x; i < ns; i += kDecodeThreads) {
      Hyps& h = H[i];
      h.nh = 1;
      h.score[0] = 0.0;
      h.ctx[0] = 0;
      h.len[0] = 0;
      h.last[0] = -1;
      h.h1[0] = 0x243f6a8885a308d3ull;
      h.h2[0] = 0x13198a2e03707344ull;
      h.p1[0] = h.p2[0] = 0;
    }
    __syncthreads();
    if (warp == 0) {
      const int R0 = beam_rows(H, ns, frame_splits + s0, 0, S.row_pe, S.row_ctx);
      if (lane == 0) S.R = R0;
    }
  }
  cluster.sync();
  const RowRes rr0{S.row_lse, S.row_l0, S.row_tl, S.row_tk};
  const RowRes rloc{S.loc_lse, S.loc_l0, S.loc_tl, S.loc_tk};
  long long ph[4] = {0, 0, 0, 0};  // thread 0: h + GEMM + push, reduce, beam step, cluster-barrier waits
  const float bias = m.out_b[c0 + (threadIdx.x & (kBcCols - 1))];  // this thread's column
  uint32_t hph = 0;  // h passes so far (the hbar phase)
  for (int32_t t = 0; t < tmax; ++t) {
    const long long ca = clock64();
    // row table from CTA 0
    if (rank != 0) {
      if (threadIdx.x == 0) S.R = S0.R;
      for (int r = threadIdx.x; r < kBcRows; r += kDecodeThreads) {
        S.row_pe[r] = S0.row_pe[r];
        S.row_ctx[r] = S0.row_ctx[r];
      }
    }
    __syncthreads();
    const int R = S.R;
    // the next frame's encoder projections (one row per live stream) into L2
    for (int i = threadIdx.x; i < ns; i += kDecodeThreads) {
      const int32_t f = frame_splits[s0 + i];
      if (t + 1 < frame_splits[s0 + i + 1] - f)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pe + static_cast<int64_t>(f + t + 1) * m.J + c0));
    }
    // h rows and this CTA's column slice of their logits, 32 rows a pass.
    // h: unit = 2 consecutive k of one row (float2 gathers, two tanhf in
    // flight); lane pairs form 4-k quads, each lane stores the quad into four
    // of the eight CTAs.  GEMM: thread = column c x group q, rows q, q+8,
    // q+16, q+24 of the pass (all 16 warps busy for R >= 8); row r's logit
    // slice goes to CTA r % 8 (local row r / 8).
    const int nloc = R > rank ? (R - rank + kBc - 1) / kBc : 0;
    if (threadIdx.x == 0) mbar_expect_tx(&S.lbar, static_cast<uint32_t>(nloc * m.Vp * 4));
    const int c = threadIdx.x & (kBcCols - 1), q = threadIdx.x / kBcCols;
    for (int p0 = 0; p0 < R; p0 += kBcPass) {
      const int Rp = min(kBcPass, R - p0);
      if (p0 > 0) cluster.sync();  // every CTA is done reading the previous pass's Hs
      if (threadIdx.x == 0) mbar_expect_tx(&S.hbar, static_cast<uint32_t>(Rp * m.J * 4));
      {
        const int half = Sl / 2, n2 = Rp * half;
        for (int base = 0; base < n2; base += kDecodeThreads) {  // uniform trip count: shuffles below
          const int x = base + threadIdx.x;
          const bool ok = x < n2;  // pairs (x, x ^ 1) are both in or both out (n2 even)
          const int lr = ok ? x / half : 0, k = rank * Sl + (x - lr * half) * 2;
          float v[2] = {0.5f, 0.5f};
          if (ok) {
            const int r = p0 + lr;
            const float2 a = *reinterpret_cast<const float2*>(pe + S.row_pe[r] * m.J + k);
            const float2 b = *reinterpret_cast<const float2*>(m.pd + static_cast<int64_t>(S.row_ctx[r]) * m.J + k);
            const float2 jb = *reinterpret_cast<const float2*>(m.j_b + k);
            v[0] = fadd(fadd(a.x, b.x), jb.x);
            v[1] = fadd(fadd(a.y, b.y), jb.y);
          }
          float z[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) z[j] = rnntg_exact::tanhf_main(v[j]);
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (!rnntg_exact::tanhf_main_path(v[j])) z[j] = rnntg_exact::tanhf_glibc(v[j]);
          const float o0 = __shfl_xor_sync(0xffffffffu, z[0], 1), o1 = __shfl_xor_sync(0xffffffffu, z[1], 1);
          if (ok) {
            const bool odd = x & 1;
            const uint32_t dst = smem_u32(Hs + lr * JS + (k & ~3)), bar = smem_u32(&S.hbar);
            const float q0 = odd ? o0 : z[0], q1 = odd ? o1 : z[1], q2 = odd ? z[0] : o0, q3 = odd ? z[1] : o1;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t d = (odd ? 4 : 0) + e;
              st_async_v4(mapa(dst, d), q0, q1, q2, q3, mapa(bar, d));
            }
          }
        }
      }
      mbar_wait(&S.hbar, hph & 1u);  // every CTA's h slices of this pass have landed
      ++hph;
      if (threadIdx.x == 0) S.stat[5] += clock64() - ca;
      const int nr = q < Rp ? (Rp - q + 7) / 8 : 0;  // rows q, q+8, ... of this pass
      if (nr > 0) {
        float acc[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = bias;
        const float* wc = Ws + c * JS;
        const float* hq = Hs + q * JS;
        if (nr == 4) logit_chain_rows<4, 2>(wc, hq, 8 * JS, m.J, acc);
        else if (nr == 3) logit_chain_rows<3, 2>(wc, hq, 8 * JS, m.J, acc);
        else if (nr == 2) logit_chain_rows<2, 4>(wc, hq, 8 * JS, m.J, acc);
        else logit_chain_rows<1, 4>(wc, hq, 8 * JS, m.J, acc);
        const int d = (p0 + q) % kBc;  // rows q + 8j all go to one CTA
        const uint32_t lb = mapa(smem_u32(&S.lbar), d);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j < nr) {
            const int r = p0 + q + 8 * j;
            st_async_b32(mapa(smem_u32(recv + (r / kBc) * m.Vp + c0 + c), d), acc[j], lb);
          }
        }
      }
    }
    const long long cb = clock64();
    if (threadIdx.x == 0) S.stat[6] += cb - ca;
    mbar_wait(&S.lbar, static_cast<uint32_t>(t & 1));  // every slice of the rows reduced here delivered
    const long long cc = clock64();
    // reduce the rows r = rank + 8 i
    double* E = reinterpret_cast<double*>(Hs);
    lse_cta_exps(recv, E, kBcPass * JS / 2, m.Vp, m.V, nloc, S.etab, S.loc_m);
    if (warp == 0) {
      lse_cta_chain(recv, E, kBcPass * JS / 2, m.Vp, m.V, nloc, S.loc_m, S.loc_lse, S.loc_l0);
    } else if (warp - 1 < nloc) {
      beam_row_reduce_n<BCAP, 1, false>(recv, m.Vp, m.V, beam, warp - 1, nloc, rloc, S.etab);
    }
    __syncthreads();
    for (int x = threadIdx.x; x < nloc * (2 + 2 * kMaxBeam); x += kDecodeThreads) {
      const int i = x / (2 + 2 * kMaxBeam), f = x - i * (2 + 2 * kMaxBeam);
      const int r = rank + kBc * i;
      if (f == 0) S0.row_lse[r] = S.loc_lse[i];
      else if (f == 1) S0.row_l0[r] = S.loc_l0[i];
      else if (f < 2 + kMaxBeam) S0.row_tl[r][f - 2] = S.loc_tl[i][f - 2];
      else S0.row_tk[r][f - 2 - kMaxBeam] = S.loc_tk[i][f - 2 - kMaxBeam];
    }
    const long long cd = clock64();
    cluster.sync();  // every row reduced
    const long long ce = clock64();
    if (rank == 0) {
      for (int i = warp; i < ns; i += kWarps) {
        const int32_t fs = frame_splits[s0 + i];
        const int32_t T = frame_splits[s0 + i + 1] - fs;
        if (t >= T) continue;
        beam_stream_step<BCAP>(m, H[i], C + static_cast<int64_t>(i) * kCandPerStream,
                               backptr + static_cast<int64_t>(fs + s0 + i) * kMaxBeam, t, T, fs, beam, merge_log,
                               length_norm, max_total, rr0, tokens, lengths + s0 + i, scores + s0 + i, &S.stat[4]);
      }
      __syncthreads();
      if (threadIdx.x == 0) S.stat[7] += clock64() - ce;  // the beam steps alone
      if (warp == 0) {
        const int Rn = beam_rows(H, ns, frame_splits + s0, t + 1, S.row_pe, S.row_ctx);
        if (lane == 0) {
          S.R = Rn;
          S.stat[1] += R;
        }
      }
    }
    const long long cf = clock64();
    cluster.sync();  // next frame's rows published
    if (threadIdx.x == 0) {
      ph[0] += cb - ca;
      ph[1] += cd - cc;
      ph[2] += cf - ce;
      ph[3] += (cc - cb) + (ce - cd) + (clock64() - cf);
    }
  }
  // Zero-frame streams: empty result, score 0.
  if (rank == 0)
    for (int i = threadIdx.x; i < ns; i += kDecodeThreads)
      if (frame_splits[s0 + i + 1] == frame_splits[s0 + i]) {
        lengths[s0 + i] = 0;
        scores[s0 + i] = 0.0;
      }
  if (rank == 0 && threadIdx.x == 0) {
    unsigned long long sf = 0;
    for (int i = 0; i < ns; ++i) sf += frame_splits[s0 + i + 1] - frame_splits[s0 + i];
    atomicAdd(&counters[0], sf);
    atomicAdd(&counters[1], S.stat[1]);
    atomicAdd(&counters[4], S.stat[4]);
    for (int i = 0; i < 4; ++i) atomicAdd(&counters[8 + i], static_cast<unsigned long long>(ph[i]));
    atomicAdd(&counters[6], S.stat[5]);  // h build (diagnostic, gather_cycles slot)
    atomicAdd(&counters[7], S.stat[7]);  // beam steps (diagnostic, gemm_wait_cycles slot)
  }
  cluster.sync();  // no CTA leaves while others may still read its shared memory
}

template <int BCAP>
size_t beam_cluster_smem(const ModelView& m, int G) {
  return static_cast<size_t>(m.J + 4) * (kBcCols + kBcPass) * 4 + static_cast<size_t>(kBcLocal) * m.Vp * 4 +
         sizeof(BcSmem) + sizeof(Hyps) * G;
}

template <int BCAP>
cudaError_t launch_beam_cluster_cap(const DecodeArgs& a, cudaStream_t s) {
  const ModelView m = view_of(*a.m);
  const int G = a.streams_per_cta;
  const int nclusters = (a.B + G - 1) / G;
  const size_t smem = beam_cluster_smem<BCAP>(m, G);
  cudaError_t e = cudaFuncSetAttribute(beam_cluster_kernel<BCAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclusters * kBc, 1, 1);
  cfg.blockDim = dim3(kDecodeThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kBc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, beam_cluster_kernel<BCAP>, m, a.pe, a.frame_splits, a.B, G, a.beam_size,
                            a.merge_op, a.length_norm, a.max_total, a.backptr, a.tokens, a.lengths, a.scores,
                            a.counters);
}

}  // namespace

int decode_num_sms_current() {
  int dev = 0;
  cudaGetDevice(&dev);
  return decode_num_sms(dev);
}

int decode_num_sms(int device) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n > 0 ? n : 1;
}

cudaError_t launch_decode_greedy(const DecodeArgs& a, cudaStream_t s) {
  const ModelView m = view_of(*a.m);
  const size_t smem = smem_common(m) + sizeof(GreedySmem);
  cudaError_t e = cudaFuncSetAttribute(
      greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
      static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int grid = (a.B + a.streams_per_cta - 1) / a.streams_per_cta;
  greedy_kernel<<<grid, kDecodeThreads, smem, s>>>(
      m, a.pe, a.frame_splits, a.B, a.streams_per_cta, std::max(1, a.symbol_cap), a.count_capped,
      a.tokens, a.lengths, a.counters);
  return cudaGetLastError();
}

namespace {
template <int BCAP, bool TC, bool SL = false>
cudaError_t launch_beam_cap3(const DecodeArgs& a, cudaStream_t s) {
  const ModelView m = view_of(*a.m);
  const int G = a.streams_per_cta;
  static const int force_r = [] {
    const char* e = std::getenv("RNNTG_DBG_FORCE_R");
    return e ? std::atoi(e) : 0;
  }();
  DbgKnobs fp{force_r};
  const size_t hl = static_cast<size_t>(hl_floats_of(m.J, m.Vp)) * 4;
  size_t smem = hl + static_cast<size_t>(2) * (TC ? 16 : kBK) * m.Vp * 4 + sizeof(BeamSmem) + sizeof(Hyps) * G +
                sizeof(BeamCand) * G * (BCAP * BCAP + 2 * BCAP);
  if (TC) smem += 1024 + static_cast<size_t>(kRowCap) * m.J * 2 + sizeof(TcBars);
  cudaError_t e = cudaFuncSetAttribute(beam_kernel<BCAP, TC, SL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int grid = (a.B + G - 1) / G;
  beam_kernel<BCAP, TC, SL><<<grid, kDecodeThreads, smem, s>>>(
      m, a.pe, a.frame_splits, a.B, G, a.beam_size, a.merge_op, a.length_norm, a.max_total,
      a.backptr, a.tokens, a.lengths, a.scores, a.counters, fp,
      BeamSlice{a.t0, a.t1, static_cast<Hyps*>(a.hyps_state)});
  return cudaGetLastError();
}

template <int BCAP, bool TC>
cudaError_t launch_beam_cap(const DecodeArgs& a, cudaStream_t s) {
  if constexpr (!TC) {
    if (a.hyps_state) return launch_beam_cap3<BCAP, false, true>(a, s);
  }
  return launch_beam_cap3<BCAP, TC>(a, s);
}

template <bool TC>
cudaError_t launch_beam_mode(const DecodeArgs& a, cudaStream_t s) {
  if (a.beam_size <= 1) return launch_beam_cap<1, TC>(a, s);
  if (a.beam_size <= 2) return launch_beam_cap<2, TC>(a, s);
  if (a.beam_size <= 4) return launch_beam_cap<4, TC>(a, s);
  return launch_beam_cap<8, TC>(a, s);
}
}  // namespace

// Hypothesis capacity is a compile-time bound (local top-k lists live in
// registers); the runtime beam_size selects the smallest capacity >= it.
// a.joiner_bf16 selects the tcgen05 joiner variant.
size_t beam_state_bytes() { return sizeof(Hyps); }

int beam_cluster_streams(const DeviceModel& d, int32_t B, int32_t beam_size, int num_sms) {
  // streams per cluster when the cluster kernel serves this batch, else 0
  if (d.Vp != kBc * kBcCols || d.V > kDecodeThreads || d.J % (4 * kBc) != 0 || B <= 0 || beam_size > kMaxBeam)
    return 0;
  // clusters that can be resident at once (8 co-scheduled SMs of one GPC each)
  static int resident = -1;
  if (resident < 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kBc * 64, 1, 1);
    cfg.blockDim = dim3(kDecodeThreads, 1, 1);
    cfg.dynamicSmemBytes = beam_cluster_smem<4>(view_of(d), 16);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kBc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaFuncSetAttribute(beam_cluster_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(cfg.dynamicSmemBytes));
    if (cudaOccupancyMaxActiveClusters(&n, beam_cluster_kernel<4>, &cfg) != cudaSuccess) n = 0;
    cudaGetLastError();
    resident = n > 0 ? n : num_sms / kBc;
  }
  const int nmax = std::min(resident, num_sms / kBc);
  // up to 14 streams a cluster (~31 joiner rows: one h / GEMM pass); beyond,
  // the second pass and the one-CTA beam steps of CTA 0 make the persistent
  // kernel as fast (measured at T = 1000, cluster vs persistent: B = 64 /
  // 128 / 160 / 192: 21.7 / 27.4 / 29.7 / 32.5 ms against 33.4 / 33.5 / - /
  // 40.5 ms; B = 240 at 16 a cluster: 40.5 against 40.2 ms)
  const int gmax = std::min(14, kBcRows / std::max(1, beam_size));
  if (B > nmax * gmax) return 0;
  const int G = (B + nmax - 1) / nmax;
  const ModelView m = view_of(d);
  const size_t smem = beam_size <= 4 ? beam_cluster_smem<4>(m, G) : beam_cluster_smem<8>(m, G);
  return smem <= 227 * 1024 ? G : 0;
}

cudaError_t launch_decode_beam_cluster(const DecodeArgs& a, cudaStream_t s) {
  if (a.beam_size <= 1) return launch_beam_cluster_cap<1>(a, s);
  if (a.beam_size <= 2) return launch_beam_cluster_cap<2>(a, s);
  if (a.beam_size <= 4) return launch_beam_cluster_cap<4>(a, s);
  return launch_beam_cluster_cap<8>(a, s);
}

cudaError_t launch_decode_beam(const DecodeArgs& a, cudaStream_t s) {
  if (a.symbol_cap > 1) {  // S > 1: sub-steps within a frame
    if (a.beam_size <= 1) return launch_beam_multi<1>(a, s);
    if (a.beam_size <= 2) return launch_beam_multi<2>(a, s);
    if (a.beam_size <= 4) return launch_beam_multi<4>(a, s);
    return launch_beam_multi<8>(a, s);
  }
  return a.joiner_bf16 ? launch_beam_mode<true>(a, s) : launch_beam_mode<false>(a, s);
}

}  // namespace rnntg
