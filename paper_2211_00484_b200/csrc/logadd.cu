// lattice_to_best_seq(lattice, kLogAdd, nbest, seed) on the device lattices
// of the last FSA decode (fsa_search.hpp:410-425):
//
//   sample_nbest (fsa.hpp:390-448): nbest paths drawn with DetRng(seed), each
//     state choosing stop / arc by the cumulative probabilities
//     exp(final - tot[s]) and exp(arc + tot[dst] - tot[s]) in arc order,
//     where tot are the log-semiring suffix totals (total_suffix_scores,
//     fsa.hpp:324-335);
//   remove_blanks_unique (fsa.hpp:452-463): blank-free label sequences in
//     first-appearance order;
//   sequence_total_logprob (fsa.hpp:533-540): per sequence, the total of the
//     lattice intersected with the sequence's blank-looped linear acceptor;
//   then the argmax by total, ties to the lexicographically smaller sequence.
//
// Every value is the reference's bit for bit: glibc's exp / log1p
// (glibc_f64.h), each state's log_add fold in its arc order, each sampling
// sum in the reference's order.  Two properties of the FSA lattices make
// the work parallel:
//  - layered: every complete path has T + 1 arcs (T frame layers and the
//    hop into the super-final node), so every sampled path consumes exactly
//    T + 2 uniforms (one per visited state) and path k's uniforms are
//    [k (T+2), (k+1)(T+2)) of the one DetRng stream: the nbest paths are
//    drawn in parallel from a pre-generated uniform sequence;
//  - node contexts: a lattice node is a (context, graph state) survivor, and
//    every path reaching it has emitted tokens ending in that context, so
//    the intersection's reachable states (node n, position i) all satisfy
//    ctx(n) == (seq[i-2], seq[i-1]).  The product DP runs over exactly those
//    cells (the reference's intersect discovers the same reachable states),
//    layer by layer, each cell's fold over its node's arcs in arc order.
#include <cstdint>

#include "decode_common.cuh"
#include "glibc_f64.h"
#include "internal.cuh"

namespace rnntg {
namespace {

struct LatArc {  // fsa.cu's lattice arc
  int32_t src, dst, label, pad;
  double score;
};

// ---------------------------------------------------------------------------
// std::mt19937_64 (the DetRng engine, common.hpp:87-127), one warp: seeding
// is sequential (lane 0), each 312-word twist runs in three parallel phases
// (words [0,156) read only old words; [156,311) read old words and the
// phase-1 results; 311 reads the new word 0), tempering per output.
// uniform01() = (x >> 11) * 2^-53.
// ---------------------------------------------------------------------------
constexpr int kMtN = 312, kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull, kMtUpper = 0xFFFFFFFF80000000ull, kMtLower = 0x7FFFFFFFull;

__device__ __forceinline__ uint64_t mt_twist1(uint64_t cur, uint64_t next, uint64_t far) {
  const uint64_t x = (cur & kMtUpper) | (next & kMtLower);
  return far ^ (x >> 1) ^ ((x & 1ull) ? kMtA : 0ull);
}
__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

__global__ void mt_uniforms_kernel(uint64_t seed, int64_t n, double* __restrict__ out) {
  __shared__ uint64_t mt[kMtN];
  const int lane = threadIdx.x;
  if (lane == 0) {
    mt[0] = seed;
    for (int i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
  }
  __syncwarp();
  for (int64_t base = 0; base < n; base += kMtN) {
    uint64_t v[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) {  // phase 1: i in [0, 156)
      const int i = lane + 32 * j;
      if (i < kMtM) v[j] = mt_twist1(mt[i], mt[i + 1], mt[i + kMtM]);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int i = lane + 32 * j;
      if (i < kMtM) mt[i] = v[j];
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 5; ++j) {  // phase 2: i in [156, 311)
      const int i = kMtM + lane + 32 * j;
      if (i < kMtN - 1) v[j] = mt_twist1(mt[i], mt[i + 1], mt[i - kMtM]);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int i = kMtM + lane + 32 * j;
      if (i < kMtN - 1) mt[i] = v[j];
    }
    __syncwarp();
    if (lane == 0) mt[kMtN - 1] = mt_twist1(mt[kMtN - 1], mt[0], mt[kMtM - 1]);
    __syncwarp();
    for (int i = lane; i < kMtN && base + i < n; i += 32)
      out[base + i] = static_cast<double>(mt_temper(mt[i]) >> 11) * 0x1.0p-53;
    __syncwarp();
  }
}

__device__ __forceinline__ uint64_t ord_of(double x) {
  const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// log_add with the shared-memory exp table (common.hpp:48-54).
__device__ __forceinline__ double ladd(double a, double b, const uint64_t* etab) {
  if (a == -INFINITY) return b;
  if (b == -INFINITY) return a;
  const double mx = a > b ? a : b, mn = a > b ? b : a;
  return rnntg_f64::xadd(mx, rnntg_f64::log1p(rnntg_f64::exp_t(rnntg_f64::xsub(mn, mx), etab)));
}

constexpr int kThreads = kLogAddWarps * 32;
constexpr int kMaxPaths = 1024;  // nbest cap of this kernel (host-checked)

struct LaSmem {
  uint64_t etab[256];
  uint64_t hash[kMaxPaths];
  int32_t plen[kMaxPaths];
  int32_t uniq[kMaxPaths];  // unique path ids in first-appearance order
  double lp[kMaxPaths];     // per unique sequence
  int32_t n_uniq;
  int32_t err;
  // per-warp layer bookkeeping of the product DP (<= kFsaMaxStates nodes a layer)
  int32_t base[kLogAddWarps][2][kFsaMaxStates + 1];
  int32_t lo[kLogAddWarps][2][kFsaMaxStates];
};

// One CTA per stream.
__global__ void __launch_bounds__(kThreads) lattice_logadd_kernel(LogAddArgs a) {
  __shared__ LaSmem S;
  const int s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  dec::load_exp_table(S.etab);
  if (threadIdx.x == 0) {
    S.n_uniq = 0;
    S.err = 0;
  }
  const int32_t fs = a.frame_splits[s];
  const int32_t T = a.frame_splits[s + 1] - fs;
  const int64_t nbase = static_cast<int64_t>(fs) * a.K + s;  // node-table base (fsa.cu's nbase)
  const int4* fi = reinterpret_cast<const int4*>(a.lat_frame_info) + (static_cast<int64_t>(fs) + s);
  const LatArc* lat = static_cast<const LatArc*>(a.lattice);
  const int32_t* nctx = a.node_ctx + nbase;
  double* tot = a.tot + nbase;
  int2* narc = a.node_arcs + nbase;
  const int32_t nn = T > 0 ? fi[T - 1].z + fi[T - 1].w : 1;  // lattice nodes; nn = super-final
  const int32_t lastb = T > 0 ? fi[T - 1].z : 0;              // layer T: the hop into the super-final
  __syncthreads();

  // ---- each node's arc range (arcs of a frame are sorted by source) ----
  for (int32_t n = threadIdx.x; n < nn; n += kThreads) narc[n] = n >= lastb ? make_int2(0, -1) : make_int2(0, 0);
  __syncthreads();
  for (int32_t t = warp; t < T; t += kLogAddWarps) {
    const int4 f = fi[t];
    for (int32_t i = lane; i < f.y; i += 32) {
      const int32_t src = lat[f.x + i].src;
      if (i == 0 || lat[f.x + i - 1].src != src) {
        int32_t e = i + 1;
        while (e < f.y && lat[f.x + e].src == src) ++e;
        narc[src] = make_int2(f.x + i, e - i);
      }
    }
  }
  __syncthreads();

  // ---- total_suffix_scores (fsa.hpp:324-335): layer by layer, backward ----
  // Layer T: -inf folded with the score-0 hop into the super-final node
  // (total 0) -> 0.  Layer t < T: the node's arcs in order.
  for (int32_t n = lastb + threadIdx.x; n < nn; n += kThreads)
    tot[n] = ladd(-INFINITY, rnntg_f64::xadd(0.0, 0.0), S.etab);
  __syncthreads();
  for (int32_t t = T - 1; t >= 0; --t) {
    const int32_t lb = t > 0 ? fi[t - 1].z : 0, ln = t > 0 ? fi[t - 1].w : 1;
    for (int32_t j = threadIdx.x; j < ln; j += kThreads) {
      const int2 r = narc[lb + j];
      double v = -INFINITY;
      for (int32_t q = 0; q < r.y; ++q) {
        const LatArc e = lat[r.x + q];
        v = ladd(v, rnntg_f64::xadd(e.score, tot[e.dst]), S.etab);
      }
      tot[lb + j] = v;
    }
    __syncthreads();
  }
  const double tot0 = tot[0];
  if (tot0 == -INFINITY) {  // no complete path: empty sequence
    if (threadIdx.x == 0) {
      a.lengths[s] = 0;
      a.logprob[s] = -INFINITY;
    }
    return;
  }

  // ---- sample_nbest (fsa.hpp:390-448): path k on its own uniforms ----
  const int64_t pstride = static_cast<int64_t>(T) + 1;
  int32_t* paths = a.paths + static_cast<int64_t>(a.nbest) * (static_cast<int64_t>(fs) + s);
  for (int k = threadIdx.x; k < a.nbest; k += kThreads) {
    const double* U = a.uniforms + static_cast<int64_t>(k) * (T + 2);
    int32_t* out = paths + k * pstride;
    int32_t len = 0, st = 0;
    uint64_t h = 0xcbf29ce484222325ull;
    for (int32_t j = 0;; ++j) {
      const double u = U[j];
      if (st == nn) break;  // super-final: stop_p = exp(0 - 0) = 1 > u
      double acc = rnntg_f64::xadd(0.0, 0.0);  // + stop_p (not final)
      const int2 r = narc[st];
      const double ts = tot[st];
      int32_t dst = nn, label = 0;
      if (r.y < 0) {  // the score-0 hop: probability exp((0 + 0) - 0) = 1
        (void)acc;
      } else {
        int32_t chosen = -1;
        for (int32_t q = 0; q < r.y; ++q) {
          const LatArc e = lat[r.x + q];
          acc = rnntg_f64::xadd(acc, rnntg_f64::exp_t(rnntg_f64::xsub(rnntg_f64::xadd(e.score, tot[e.dst]), ts),
                                                      S.etab));
          if (u < acc) {
            chosen = q;
            break;
          }
        }
        if (chosen < 0)  // rounding left u past the last bucket: the last live arc
          for (int32_t q = r.y - 1; q >= 0; --q) {
            const LatArc e = lat[r.x + q];
            if (rnntg_f64::xadd(e.score, tot[e.dst]) != -INFINITY) {
              chosen = q;
              break;
            }
          }
        if (chosen < 0) break;  // (cannot happen on a live state)
        const LatArc e = lat[r.x + chosen];
        dst = e.dst;
        label = e.label;
      }
      if (label != 0) {
        out[len++] = label;
        h = (h ^ static_cast<uint64_t>(label)) * 0x100000001b3ull;
      }
      st = dst;
    }
    S.plen[k] = len;
    S.hash[k] = h ^ static_cast<uint64_t>(len);
  }
  __syncthreads();

  // ---- remove_blanks_unique: first appearances, in order ----
  for (int k0 = 0; k0 < a.nbest; k0 += kThreads) {
    const int k = k0 + threadIdx.x;
    bool first = k < a.nbest;
    for (int j = 0; first && j < k; ++j) {
      if (S.hash[j] != S.hash[k] || S.plen[j] != S.plen[k]) continue;
      const int32_t* x = paths + k * pstride;
      const int32_t* y = paths + j * pstride;
      bool same = true;
      for (int32_t q = 0; same && q < S.plen[k]; ++q) same = x[q] == y[q];
      if (same) first = false;
    }
    // block-wide ordered compaction of this round
    const unsigned bal = __ballot_sync(0xffffffffu, first);
    __shared__ int32_t wcount[kLogAddWarps];
    if (lane == 0) wcount[warp] = __popc(bal);
    __syncthreads();
    int off = S.n_uniq;
    for (int w = 0; w < warp; ++w) off += wcount[w];
    if (first) S.uniq[off + __popc(bal & ((1u << lane) - 1u))] = k;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 0; w < kLogAddWarps; ++w) S.n_uniq += wcount[w];
    __syncthreads();
  }
  const int nu = S.n_uniq;

  // ---- sequence_total_logprob per unique sequence (warp per sequence) ----
  const int V = a.V;
  const int64_t gw = static_cast<int64_t>(s) * kLogAddWarps + warp;
  double* cellbuf = a.cells + gw * 2 * a.cell_cap;
  int32_t* skey = a.pos + gw * 3 * (a.tmax + 2);
  int32_t* spos = skey + (a.tmax + 2);
  int32_t* rrank = spos + (a.tmax + 2);
  for (int qu = warp; qu < nu; qu += kLogAddWarps) {
    const int32_t* seq = paths + S.uniq[qu] * pstride;
    const int32_t L = S.plen[S.uniq[qu]];
    auto ctx_at = [&](int32_t i) {
      const int32_t x = i >= 2 ? seq[i - 2] : 0, y = i >= 1 ? seq[i - 1] : 0;
      return x * V + y;
    };
    // positions 0..L sorted by context: rank = #smaller keys + #equal keys before
    for (int32_t i = lane; i <= L; i += 32) {
      const int32_t c = ctx_at(i);
      int32_t less = 0, eq = 0;
      for (int32_t j = 0; j <= L; ++j) {
        const int32_t cj = ctx_at(j);
        less += cj < c ? 1 : 0;
        eq += (cj == c && j < i) ? 1 : 0;
      }
      skey[less + eq] = c;
      spos[less + eq] = i;
      rrank[i] = eq;
    }
    __syncwarp();
    // cells of a layer: node j's cells are its context's positions, at
    // base[j] + (rank of the position among equal contexts)
    auto layer_setup = [&](int32_t lb, int32_t ln, int bsel) -> int32_t {
      int32_t run = 0;
      for (int32_t j0 = 0; j0 < ln; j0 += 32) {
        const int32_t j = j0 + lane;
        int32_t cnt = 0, lo = 0;
        if (j < ln) {
          const int32_t c = nctx[lb + j];
          int32_t a0 = 0, a1 = L + 1;  // first key >= c
          while (a0 < a1) {
            const int32_t mid = (a0 + a1) >> 1;
            if (skey[mid] < c) a0 = mid + 1;
            else a1 = mid;
          }
          lo = a0;
          int32_t b0 = a0, b1 = L + 1;  // first key > c
          while (b0 < b1) {
            const int32_t mid = (b0 + b1) >> 1;
            if (skey[mid] <= c) b0 = mid + 1;
            else b1 = mid;
          }
          cnt = b0 - a0;
        }
        int32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t x = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += x;
        }
        if (j < ln) {
          S.base[warp][bsel][j] = run + incl - cnt;
          S.lo[warp][bsel][j] = lo;
        }
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) S.base[warp][bsel][ln] = run;
      __syncwarp();
      return run;
    };
    // layer T (nodes [lastb, nn)): the score-0 hop into the super-final,
    // whose one final cell is (sf, L) with total 0 + 0.
    int cur = 0;
    int32_t ncells = layer_setup(lastb, nn - lastb, cur);
    if (ncells > a.cell_cap) {
      if (lane == 0) atomicExch(a.error_flag, 1);
      break;
    }
    for (int32_t c = lane; c < ncells; c += 32) {
      int32_t j = 0;
      while (S.base[warp][cur][j + 1] <= c) ++j;
      const int32_t i = spos[S.lo[warp][cur][j] + c - S.base[warp][cur][j]];
      const double hop = rnntg_f64::xadd(rnntg_f64::xadd(0.0, 0.0), i == L ? rnntg_f64::xadd(0.0, 0.0) : -INFINITY);
      cellbuf[cur * a.cell_cap + c] = ladd(-INFINITY, hop, S.etab);
    }
    __syncwarp();
    bool overflow = false;
    for (int32_t t = T - 1; t >= 0; --t) {
      const int32_t nb1 = fi[t].z;  // layer t+1 base node
      const int32_t lb = t > 0 ? fi[t - 1].z : 0, ln = t > 0 ? fi[t - 1].w : 1;
      const int nxt = cur ^ 1;
      ncells = layer_setup(lb, ln, nxt);
      if (ncells > a.cell_cap) {
        overflow = true;
        break;
      }
      const double* up = cellbuf + cur * a.cell_cap;
      for (int32_t c = lane; c < ncells; c += 32) {
        int32_t j = 0;
        while (S.base[warp][nxt][j + 1] <= c) ++j;
        const int32_t i = spos[S.lo[warp][nxt][j] + c - S.base[warp][nxt][j]];
        const int2 r = narc[lb + j];
        double v = -INFINITY;
        for (int32_t q = 0; q < r.y; ++q) {
          const LatArc e = lat[r.x + q];
          int32_t i2;
          if (e.label == 0) i2 = i;
          else if (i < L && e.label == seq[i]) i2 = i + 1;
          else continue;
          const int32_t d = e.dst - nb1;
          const double sv = up[S.base[warp][cur][d] + rrank[i2]];
          v = ladd(v, rnntg_f64::xadd(rnntg_f64::xadd(e.score, 0.0), sv), S.etab);
        }
        cellbuf[nxt * a.cell_cap + c] = v;
      }
      __syncwarp();
      cur = nxt;
    }
    if (overflow) {
      if (lane == 0) atomicExch(a.error_flag, 1);
      break;
    }
    // the start state (node 0, position 0): node 0's only cell
    if (lane == 0) S.lp[qu] = cellbuf[cur * a.cell_cap + S.base[warp][cur][0] + rrank[0]];
    __syncwarp();
  }
  __syncthreads();

  // ---- argmax by total, ties to the lexicographically smaller sequence ----
  if (threadIdx.x == 0) {
    int best = -1;
    double best_lp = -INFINITY;
    for (int qu = 0; qu < nu; ++qu) {
      const double lp = S.lp[qu];
      bool take = best < 0 || lp > best_lp;
      if (!take && lp == best_lp) {  // std::vector operator<
        const int32_t* x = paths + S.uniq[qu] * pstride;
        const int32_t* y = paths + S.uniq[best] * pstride;
        const int32_t lx = S.plen[S.uniq[qu]], ly = S.plen[S.uniq[best]];
        int32_t q = 0;
        while (q < lx && q < ly && x[q] == y[q]) ++q;
        take = q < lx && q < ly ? x[q] < y[q] : lx < ly;
      }
      if (take) {
        best = qu;
        best_lp = lp;
      }
    }
    const int32_t* x = paths + S.uniq[best] * pstride;
    const int32_t len = S.plen[S.uniq[best]];
    for (int32_t q = 0; q < len; ++q) a.tokens[fs + q] = x[q];
    a.lengths[s] = len;
    a.logprob[s] = best_lp;
  }
}

}  // namespace

cudaError_t launch_mt19937_64_uniforms(uint64_t seed, int64_t n, double* out, cudaStream_t s) {
  mt_uniforms_kernel<<<1, 32, 0, s>>>(seed, n, out);
  return cudaGetLastError();
}

cudaError_t launch_lattice_logadd(const LogAddArgs& a, cudaStream_t s) {
  if (a.B <= 0) return cudaSuccess;
  if (a.nbest > kMaxPaths) return cudaErrorInvalidValue;
  lattice_logadd_kernel<<<a.B, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rnntg
