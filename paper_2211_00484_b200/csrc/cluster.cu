// Small-batch greedy on thread-block clusters (greedy_search_batch,
// search.hpp:107-167, S = 1).
//
// With few streams the persistent kernel of decode.cu leaves most SMs idle
// and each busy SM streams all of out_w (1 MB) from L2 every frame for a
// handful of joiner rows, so a frame costs ~20 us regardless of the row
// count.  Here a cluster of kCl = 8 CTAs serves up to 8 streams: CTA c keeps
// the out_w columns [c*CW, (c+1)*CW) (CW = Vp/8) resident in shared memory
// for the whole utterance, every CTA builds the h rows of the cluster's
// streams, computes its column slice of the logits (sequential FMUL/FADD per
// column, the reference's order), and posts its slice's first-max (value,
// index) into every CTA's shared memory (DSMEM, frame-parity buffered).
// After ONE cluster barrier per frame each CTA combines the 8 partials in
// rank order with the same first-max rule (search.hpp:61-66) and advances its
// own copy of the contexts (identical in all CTAs); CTA 0 appends the
// non-blank tokens.  The next frame's pe rows are fetched with cp.async while
// the logits run, and a stream's pd[ctx] row is cached in shared memory until
// its context moves (blank frames, the common case, reload nothing).  No
// weight traffic after the first frame.
#include <cooperative_groups.h>
#include <float.h>

#include "decode_common.cuh"

namespace cg = cooperative_groups;

namespace rnntg {
namespace {

using namespace dec;

constexpr int kCl = 8;          // CTAs per cluster (portable maximum)
constexpr int kClThreads = 256;
constexpr int kClRows = 8;      // streams per cluster

struct ClSmem {
  uint64_t xbar[2];  // per frame parity: every CTA's slice maxima of the frame have landed
  uint64_t hbar[2];  // per frame parity: every CTA's h slices of the frame have landed
  uint2 part[2][kCl][kClRows];  // per frame parity, rank, row: slice first-max (value bits, index)
  int32_t ctx[kClRows];     // per stream slot; every CTA keeps an identical copy
  int32_t len[kClRows];
  int32_t nfr[kClRows];     // frames of the slot's stream
  int32_t fs[kClRows];      // its first frame
  int32_t pd_ctx[kClRows];  // context whose pd slice PdS[i] holds (-1: none)
  int32_t spec_t[kClRows];  // frame whose h row of slot i was built ahead, with
  int32_t spec_ctx[kClRows];  //   context spec_ctx[i]
  int32_t row_s[kClRows];   // this frame: compact row -> stream slot
  int32_t rb[kClRows];      // this frame: compact rows rebuilt (into Hr)
  int32_t rbflag[kClRows];  // this frame: row r reads Hr (else Hs[parity])
  int32_t nrow_s[kClRows];  // next frame: compact row -> stream slot
  int32_t nrb, nR, nsp;
  long long chain_clk;      // thread 0: the logit chain part of the GEMM phase
};

// Shared memory of one CTA: out_w slice, two frames of h rows plus the
// rebuilt rows, this CTA's k-slice of two frames of pe rows, of the slots'
// pd rows and of j_b, then the ClSmem block.
__host__ __device__ constexpr size_t cluster_smem_bytes(int J, int Vp) {
  return (static_cast<size_t>(J + 4) * (Vp / kCl + 3 * kClRows) + static_cast<size_t>(3 * kClRows + 1) * (J / kCl)) *
             4 +
         sizeof(ClSmem);
}

// The cluster builds each h row tanhf((pe + pd[ctx]) + j_b) together: CTA
// `rank` evaluates k in [rank*Sl, (rank+1)*Sl) (Sl = J/8; glibc-exact tanhf,
// branch-free main path, special inputs fixed up) and stores the slice into
// row r of `dst` in every CTA of the cluster, completing J*4 bytes per row on
// each receiver's `bar`.  List entry q names compact row r = rows ? rows[q]
// : q of stream slot row_s[r]; tid/nt enumerate whole warps.
__device__ __noinline__ void build_send_h(float* dst, uint64_t* bar, int JS, const float* PeS,
                                             const float* PdS, const float* JbS, int Sl, int rank,
                                             const int32_t* rows, const int32_t* row_s, int nq, int tid,
                                             int nt) {
  const int n = nq * Sl;
  const int lane = tid & 31;
  for (int base = 0; base < n; base += nt) {
    const int x = base + tid;
    const bool ok = x < n;
    const int q = ok ? x / Sl : 0, j = x - q * Sl;
    const int r = rows ? rows[q] : q;
    const int i = row_s[r];
    const float v = ok ? fadd(fadd(PeS[i * Sl + j], PdS[i * Sl + j]), JbS[j]) : 0.5f;
    float z = rnntg_exact::tanhf_main(v);
    if (!rnntg_exact::tanhf_main_path(v)) z = rnntg_exact::tanhf_glibc(v);
    // lanes 4g..4g+3 hold 4 consecutive k of one row (Sl % 4 == 0): each
    // sends the quad to two of the eight CTAs
    const int g = lane & ~3;
    const float z0 = __shfl_sync(0xffffffffu, z, g), z1 = __shfl_sync(0xffffffffu, z, g + 1);
    const float z2 = __shfl_sync(0xffffffffu, z, g + 2), z3 = __shfl_sync(0xffffffffu, z, g + 3);
    if (ok) {
      const uint32_t a = smem_u32(dst + r * JS + rank * Sl + (j & ~3)), ba = smem_u32(bar);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint32_t d = 2 * (lane & 3) + e;
        st_async_v4(mapa(a, d), z0, z1, z2, z3, mapa(ba, d));
      }
    }
  }
}

// acc[r] += w[k] * h_r[k] for k = 0..J-1 in order (FMUL, then FADD: the
// reference's sequential sum), NR rows sharing the column.  The operands of
// the next 16 k are loaded while the current 16 run, so the shared-memory
// latency stays under the dependent FADD chain.  J % 16 == 0.
template <int NR>
__device__ __forceinline__ void logit_chain(const float* wc, const float* ha, const float* hb, int J,
                                            float* acc) {
  constexpr int U = 4;  // float4 per block
  float4 w[U], a[U], b[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    w[u] = *reinterpret_cast<const float4*>(wc + 4 * u);
    a[u] = *reinterpret_cast<const float4*>(ha + 4 * u);
    if (NR == 2) b[u] = *reinterpret_cast<const float4*>(hb + 4 * u);
  }
  for (int k = 0; k < J; k += 4 * U) {
    const int kn = min(k + 4 * U, J - 4 * U);  // the last block reloads itself
    float4 wn[U], an[U], bn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      wn[u] = *reinterpret_cast<const float4*>(wc + kn + 4 * u);
      an[u] = *reinterpret_cast<const float4*>(ha + kn + 4 * u);
      if (NR == 2) bn[u] = *reinterpret_cast<const float4*>(hb + kn + 4 * u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc[0] = fadd(acc[0], fmul(w[u].x, a[u].x));
      if (NR == 2) acc[1] = fadd(acc[1], fmul(w[u].x, b[u].x));
      acc[0] = fadd(acc[0], fmul(w[u].y, a[u].y));
      if (NR == 2) acc[1] = fadd(acc[1], fmul(w[u].y, b[u].y));
      acc[0] = fadd(acc[0], fmul(w[u].z, a[u].z));
      if (NR == 2) acc[1] = fadd(acc[1], fmul(w[u].z, b[u].z));
      acc[0] = fadd(acc[0], fmul(w[u].w, a[u].w));
      if (NR == 2) acc[1] = fadd(acc[1], fmul(w[u].w, b[u].w));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      w[u] = wn[u];
      a[u] = an[u];
      if (NR == 2) b[u] = bn[u];
    }
  }
}

__global__ void __launch_bounds__(kClThreads, 1)
    greedy_cluster_kernel(ModelView m, const float* __restrict__ pe,
                          const int32_t* __restrict__ frame_splits, int32_t B, int32_t G,
                          int32_t* __restrict__ tokens, int32_t* __restrict__ lengths,
                          unsigned long long* __restrict__ counters) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int cl = blockIdx.x / kCl;
  const int CW = m.Vp / kCl;
  const int J = m.J;
  const int Sl = J / kCl;  // this CTA's k-slice of the h rows: [rank*Sl, (rank+1)*Sl)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // Column-major slices, k contiguous: a thread's column (and a row of h)
  // is read 4 k at a time (LDS.128); the +4 pad spreads the 64 columns'
  // 16-byte reads over distinct banks.
  const int JS = J + 4;
  float* Ws = reinterpret_cast<float*>(smem_raw);  // [CW][J+4] out_w slice
  float* Hs = Ws + CW * JS;                        // [2][kClRows][J+4] h rows built ahead, by frame parity
  float* Hr = Hs + 2 * kClRows * JS;               // [kClRows][J+4] h rows rebuilt this frame
  float* PeS = Hr + kClRows * JS;                  // [2][kClRows][Sl] pe slices, by frame parity
  float* PdS = PeS + 2 * kClRows * Sl;             // [kClRows][Sl] pd[ctx] slices (cached)
  float* JbS = PdS + kClRows * Sl;                 // [Sl]
  ClSmem& S = *reinterpret_cast<ClSmem*>(JbS + Sl);

  const int s0 = cl * G;
  const int ns = max(0, min(G, B - s0));
  const int c0 = rank * CW;
  for (int x = threadIdx.x; x < J * CW; x += kClThreads) {
    const int k = x / CW, c = x - k * CW;
    Ws[c * JS + k] = m.out_wt[static_cast<int64_t>(k) * m.Vp + c0 + c];
  }
  for (int j = threadIdx.x; j < Sl; j += kClThreads) JbS[j] = m.j_b[rank * Sl + j];
  if (threadIdx.x == 0) {
    S.chain_clk = 0;
    for (int p = 0; p < 2; ++p) {
      mbar_init(&S.xbar[p], 1);
      mbar_init(&S.hbar[p], 1);
    }
    fence_mbar_init();
  }
  if (threadIdx.x < kClRows) {
    const int i = threadIdx.x;
    S.ctx[i] = 0;
    S.len[i] = 0;
    S.pd_ctx[i] = -1;
    S.spec_t[i] = -1;
    S.fs[i] = i < ns ? frame_splits[s0 + i] : 0;
    S.nfr[i] = i < ns ? frame_splits[s0 + i + 1] - frame_splits[s0 + i] : 0;
  }
  __syncthreads();
  int32_t tmax = 0, nfr_r[kClRows];
#pragma unroll
  for (int i = 0; i < kClRows; ++i) {
    nfr_r[i] = S.nfr[i];  // 0 past ns
    tmax = max(tmax, nfr_r[i]);
  }
  // Asynchronous fetches of this CTA's slices: pe rows of frame t for the
  // slots live at t (into PeS[t & 1]), pd[ctx] for the slots whose context
  // moved.  Waited for at the top of the frame that reads them.
  const int Sl4 = Sl / 4;
  auto fetch_pe = [&](int32_t t, int tid, int nt) {
    float* P = PeS + (t & 1) * kClRows * Sl;
    for (int x = tid; x < ns * Sl4; x += nt) {
      const int i = x / Sl4, j = (x - i * Sl4) * 4;
      if (t < S.nfr[i]) cp_async16(P + i * Sl + j, pe + static_cast<int64_t>(S.fs[i] + t) * J + rank * Sl + j);
    }
    cp_async_commit();
  };
  auto fetch_pd = [&]() {
    for (int x = kClThreads - 1 - threadIdx.x; x < ns * Sl4; x += kClThreads) {
      const int i = x / Sl4, j = (x - i * Sl4) * 4;
      if (S.pd_ctx[i] != S.ctx[i])
        cp_async16(PdS + i * Sl + j, m.pd + static_cast<int64_t>(S.ctx[i]) * J + rank * Sl + j);
    }
    cp_async_commit();
  };
  fetch_pe(0, threadIdx.x, kClThreads);
  fetch_pe(1, threadIdx.x, kClThreads);
  fetch_pd();
  const float bias = threadIdx.x % 64 < CW ? m.out_b[c0 + threadIdx.x % 64] : 0.0f;  // this thread's column
  cluster.sync();  // barriers initialised cluster-wide before any remote store
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long rows_total = 0;

  long long ph[4] = {0, 0, 0, 0};  // thread 0: h rows, logits + slice max, slice exchange, combine
  long long spec_clk = 0;          // first worker thread: fetch + h rows ahead
  for (int32_t t = 0; t < tmax; ++t) {
    const long long ca = clock64();
    const int par = t & 1;
    // rows of the live streams (compact, stream order); the ones not built
    // ahead with the current context (rebuilt now); next frame's rows.
    // Warp 0, lane i = slot i, compacts them with ballots.
    int R = 0;
#pragma unroll
    for (int i = 0; i < kClRows; ++i) R += t < nfr_r[i];
    if (warp == 0) {
      const int i = lane;
      const bool live = i < ns && t < S.nfr[i];
      const bool ahead = live && S.spec_t[i] == t;
      const bool rebuild = live && !(ahead && S.spec_ctx[i] == S.ctx[i]);
      const bool nlive = i < ns && t + 1 < S.nfr[i];
      const unsigned lt = (1u << lane) - 1u;
      const unsigned mlive = __ballot_sync(0xffffffffu, live), mrb = __ballot_sync(0xffffffffu, rebuild);
      const unsigned mnext = __ballot_sync(0xffffffffu, nlive), mahead = __ballot_sync(0xffffffffu, ahead);
      if (live) {
        const int r = __popc(mlive & lt);
        S.row_s[r] = i;
        S.rbflag[r] = rebuild;
        if (rebuild) S.rb[__popc(mrb & lt)] = r;
      }
      if (nlive) S.nrow_s[__popc(mnext & lt)] = i;
      if (lane == 0) {
        S.nrb = __popc(mrb);
        S.nR = __popc(mnext);
        S.nsp = __popc(mahead);
      }
    }
    rows_total += R;
    cp_async_wait_all();
    __syncthreads();
    if (threadIdx.x < ns) S.pd_ctx[threadIdx.x] = S.ctx[threadIdx.x];
    if (threadIdx.x == (R == 1 ? 128 : kClThreads - 32)) {
      // this frame's deliveries (armed off thread 0's path, by a warp with no
      // logit rows when R = 1): rows built ahead (sent last frame) and rows
      // rebuilt now, J*4 bytes each; R slice maxima from each CTA
      mbar_expect_tx(&S.hbar[par], static_cast<uint32_t>((S.nsp + S.nrb) * J * 4));
      mbar_expect_tx(&S.xbar[par], static_cast<uint32_t>(R * kCl * sizeof(uint2)));
    }
    const int nrb = S.nrb;
    if (nrb > 0) {
      build_send_h(Hr, &S.hbar[par], JS, PeS + par * kClRows * Sl, PdS, JbS, Sl, rank, S.rb, S.row_s, nrb,
                   threadIdx.x, kClThreads);
      __syncthreads();  // PeS[par] is read: free for frame t + 2
    }
    const long long cb = clock64();
    // Warps without logit rows this frame (on the SM sub-partitions the
    // chain warps leave free when R = 1) fetch frame t + 2's pe slices and
    // build frame t + 1's h rows ahead, assuming every stream's context
    // stays (a blank: most frames).  A stream that emits is rebuilt at the
    // top of the next frame.
    const int busy = 2 * min(R, 4);
    int widx = -1, nw = 0;
    if (R == 1) {
      nw = 128;
      if (warp >= 2 && (warp & 3) >= 2) widx = ((warp >> 2) * 2 + (warp & 3) - 2) * 32 + lane;
    } else if (busy < 8) {
      nw = (8 - busy) * 32;
      if (warp >= busy) widx = threadIdx.x - busy * 32;
    }
    if (nw == 0) fetch_pe(t + 2, threadIdx.x, kClThreads);
    // logits of this CTA's columns: thread = (column c, row slot q), rows q, q+4
    {
      const int c = threadIdx.x % 64, q = threadIdx.x / 64;
      const bool cok = c < CW && c0 + c < m.V;
      float acc[2];
      acc[0] = acc[1] = bias;
      if (widx >= 0) {
        fetch_pe(t + 2, widx, nw);
        const int nR = S.nR;
        if (nR > 0) {
          build_send_h(Hs + (par ^ 1) * kClRows * JS, &S.hbar[par ^ 1], JS, PeS + (par ^ 1) * kClRows * Sl, PdS,
                       JbS, Sl, rank, nullptr, S.nrow_s, nR, widx, nw);
          if (widx < nR) {
            const int i = S.nrow_s[widx];
            S.spec_t[i] = t + 1;
            S.spec_ctx[i] = S.ctx[i];
          }
        }
        if (widx == 0) spec_clk += clock64() - cb;
      } else if (c < CW && q < R) {
        mbar_wait(&S.hbar[par], (t >> 1) & 1);  // every CTA's h slices of this frame have landed
        const float* HsCur = Hs + par * kClRows * JS;
        const float* ha = (S.rbflag[q] ? Hr : HsCur) + q * JS;
        // The sum is one 512-long dependent FADD chain per logit, k in
        // order; operands come 4 k per 16-byte load.
        const float* wc = Ws + c * JS;
        if (q + 4 < R)
          logit_chain<2>(wc, ha, (S.rbflag[q + 4] ? Hr : HsCur) + (q + 4) * JS, J, acc);
        else
          logit_chain<1>(wc, ha, ha, J, acc);
      }
      if (threadIdx.x == 0) S.chain_clk += clock64() - cb;
      // slice first-max per row: 64 threads (2 warps) per row slot; the
      // result goes to every CTA of the cluster (st.async into DSMEM,
      // frame-parity buffered), so each CTA combines the slices itself
      const int nu = R > 4 ? 2 : 1;
      for (int u = 0; u < nu; ++u) {
        const int r = q + 4 * u;
        float bv = (cok && r < R) ? acc[u] : -FLT_MAX;
        int bk = (cok && r < R) ? c0 + c : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
          if (tok_before(ov, ok, bv, bk)) {
            bv = ov;
            bk = ok;
          }
        }
        __shared__ float wv[8][2];
        __shared__ int wk[8][2];
        if (lane == 0) {
          wv[r & 7][warp & 1] = bv;
          wk[r & 7][warp & 1] = bk;
        }
        __syncthreads();
        if ((warp & 1) == 0 && r < R && lane < kCl) {
          float v = wv[r][0];
          int k = wk[r][0];
          if (tok_before(wv[r][1], wk[r][1], v, k)) {
            v = wv[r][1];
            k = wk[r][1];
          }
          st_async_v2(mapa(smem_u32(&S.part[par][rank][r]), lane), __float_as_uint(v), static_cast<uint32_t>(k),
                      mapa(smem_u32(&S.xbar[par]), lane));
        }
        if (u + 1 < nu) __syncthreads();
      }
    }
    const long long cc = clock64();
    long long cd = cc;
    if (threadIdx.x < R) {
      mbar_wait(&S.xbar[par], (t >> 1) & 1);  // every slice of this frame has landed
      cd = clock64();
      const int r = threadIdx.x;
      float bv = -FLT_MAX;
      int bk = 0x7fffffff;
      for (int c = 0; c < kCl; ++c) {
        const uint2 e = S.part[par][c][r];
        if (tok_before(__uint_as_float(e.x), static_cast<int>(e.y), bv, bk)) {
          bv = __uint_as_float(e.x);
          bk = static_cast<int>(e.y);
        }
      }
      const int i = S.row_s[r];
      if (bk != 0) {
        const int32_t len = S.len[i];
        if (rank == 0) tokens[S.fs[i] + len] = bk;
        S.len[i] = len + 1;
        S.ctx[i] = (S.ctx[i] % m.V) * m.V + bk;
      }
    }
    __syncthreads();
    fetch_pd();
    if (threadIdx.x == 0) {
      const long long ce = clock64();
      ph[0] += cb - ca;
      ph[1] += cc - cb;
      ph[2] += cd - cc;
      ph[3] += ce - cd;
    }
  }
  cp_async_wait_all();
  if (rank == 0 && threadIdx.x < ns) lengths[s0 + threadIdx.x] = S.len[threadIdx.x];
  if (rank == 0 && threadIdx.x == 0) {
    unsigned long long sf = 0;
    for (int i = 0; i < ns; ++i) sf += S.nfr[i];
    atomicAdd(&counters[0], sf);
    atomicAdd(&counters[1], rows_total);
    for (int i = 0; i < 4; ++i) atomicAdd(&counters[8 + i], static_cast<unsigned long long>(ph[i]));
    atomicAdd(&counters[6], static_cast<unsigned long long>(S.chain_clk));
  }
  if (rank == 0 && spec_clk > 0) atomicAdd(&counters[7], static_cast<unsigned long long>(spec_clk));
  cluster.sync();  // no CTA leaves while others may still write its shared memory
}

}  // namespace

bool greedy_cluster_fits(const DeviceModel& d, int32_t B) {
  return B > 0 && B <= 18 * kClRows && d.Vp % kCl == 0 && d.J % 32 == 0 &&
         cluster_smem_bytes(d.J, d.Vp) <= 226 * 1024;
}

cudaError_t launch_decode_greedy_cluster(const DecodeArgs& a, cudaStream_t s) {
  const ModelView m = view_of(*a.m);
  // one stream per cluster up to 18 clusters (144 SMs), then up to 8 each
  const int nclusters = std::max((a.B + kClRows - 1) / kClRows, std::min(18, a.B));
  const int G = (a.B + nclusters - 1) / nclusters;
  const size_t smem = cluster_smem_bytes(m.J, m.Vp);
  cudaError_t e = cudaFuncSetAttribute(greedy_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclusters * kCl, 1, 1);
  cfg.blockDim = dim3(kClThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, greedy_cluster_kernel, m, a.pe, a.frame_splits, a.B, G, a.tokens, a.lengths,
                            a.counters);
}

}  // namespace rnntg
