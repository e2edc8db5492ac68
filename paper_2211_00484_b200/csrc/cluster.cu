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
// index) into CTA 0's shared memory (DSMEM).  After a cluster barrier CTA 0
// combines the 8 partials in rank order with the same first-max rule
// (search.hpp:61-66), appends non-blank tokens, advances the contexts and
// publishes them; every CTA reads them back through DSMEM.  Two cluster
// barriers per frame; no weight traffic after the first frame.
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
  float part_v[kCl][kClRows];   // CTA 0: per-rank slice maxima
  int32_t part_k[kCl][kClRows];
  int32_t ctx[kClRows];         // CTA 0: authoritative contexts; others: copies
  int32_t len[kClRows];
  int64_t row_pe[kClRows];
  int32_t row_ctx[kClRows];
  int32_t live[kClRows];
};

__global__ void __launch_bounds__(kClThreads, 1)
    greedy_cluster_kernel(ModelView m, const float* __restrict__ pe,
                          const int32_t* __restrict__ frame_splits, int32_t B, int32_t G,
                          int32_t* __restrict__ tokens, int32_t* __restrict__ lengths,
                          unsigned long long* __restrict__ counters) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int cl = blockIdx.x / kCl;
  const int CW = m.Vp / kCl;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* Ws = reinterpret_cast<float*>(smem_raw);  // [J][CW] k-major out_w slice
  float* Hs = Ws + m.J * CW;                       // [J][kClRows] k-major h rows
  ClSmem& S = *reinterpret_cast<ClSmem*>(Hs + m.J * kClRows);
  ClSmem& S0 = *cluster.map_shared_rank(&S, 0);

  const int s0 = cl * G;
  const int ns = max(0, min(G, B - s0));
  const int c0 = rank * CW;
  for (int x = threadIdx.x; x < m.J * CW; x += kClThreads) {
    const int k = x / CW, c = x - k * CW;
    Ws[x] = m.out_wt[static_cast<int64_t>(k) * m.Vp + c0 + c];
  }
  if (threadIdx.x < kClRows) {
    S.ctx[threadIdx.x] = 0;
    S.len[threadIdx.x] = 0;
  }
  int32_t tmax = 0;
  for (int i = 0; i < ns; ++i) tmax = max(tmax, frame_splits[s0 + i + 1] - frame_splits[s0 + i]);
  cluster.sync();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long rows_total = 0;

  for (int32_t t = 0; t < tmax; ++t) {
    // rows of the live streams (compact, stream order)
    if (threadIdx.x == 0) {
      int R = 0;
      for (int i = 0; i < ns; ++i) {
        const int32_t fs = frame_splits[s0 + i];
        S.live[i] = t < frame_splits[s0 + i + 1] - fs;
        if (S.live[i]) {
          S.row_pe[R] = fs + t;
          S.row_ctx[R] = S.ctx[i];
          ++R;
        }
      }
    }
    __syncthreads();
    int R = 0;
    for (int i = 0; i < ns; ++i) R += S.live[i];
    rows_total += R;
    // h rows: tanhf((pe + pd[ctx]) + j_b), glibc-exact
    for (int x = threadIdx.x; x < R * m.J; x += kClThreads) {
      const int r = x / m.J, k = x - r * m.J;
      const float a = pe[S.row_pe[r] * m.J + k];
      const float b = m.pd[static_cast<int64_t>(S.row_ctx[r]) * m.J + k];
      const float v = fadd(fadd(a, b), m.j_b[k]);
      Hs[k * kClRows + r] = rnntg_exact::tanhf_glibc(v);
    }
    __syncthreads();
    // logits of this CTA's columns: thread = (column c, row slot q), rows q, q+4
    {
      const int c = threadIdx.x % 64, q = threadIdx.x / 64;
      const bool cok = c < CW && c0 + c < m.V;
      float acc[2];
      const float bias = c < CW ? m.out_b[c0 + c] : 0.0f;
      acc[0] = acc[1] = bias;
      if (c < CW) {
        if (q + 4 < R) {
          for (int k = 0; k < m.J; ++k) {
            const float w = Ws[k * CW + c];
            acc[0] = fadd(acc[0], fmul(w, Hs[k * kClRows + q]));
            acc[1] = fadd(acc[1], fmul(w, Hs[k * kClRows + q + 4]));
          }
        } else if (q < R) {
          for (int k = 0; k < m.J; ++k) acc[0] = fadd(acc[0], fmul(Ws[k * CW + c], Hs[k * kClRows + q]));
        }
      }
      // slice first-max per row: 64 threads (2 warps) per row slot
#pragma unroll
      for (int u = 0; u < 2; ++u) {
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
        // two warps per row slot: combine through CTA 0's partial table
        __shared__ float wv[8][2];
        __shared__ int wk[8][2];
        if (lane == 0) {
          wv[r & 7][warp & 1] = bv;
          wk[r & 7][warp & 1] = bk;
        }
        __syncthreads();
        if (lane == 0 && (warp & 1) == 0 && r < R) {
          float v = wv[r][0];
          int k = wk[r][0];
          if (tok_before(wv[r][1], wk[r][1], v, k)) {
            v = wv[r][1];
            k = wk[r][1];
          }
          S0.part_v[rank][r] = v;
          S0.part_k[rank][r] = k;
        }
        __syncthreads();
      }
    }
    cluster.sync();  // partials posted
    if (rank == 0 && threadIdx.x < R) {
      const int r = threadIdx.x;
      float bv = -FLT_MAX;
      int bk = 0x7fffffff;
      for (int c = 0; c < kCl; ++c)
        if (tok_before(S.part_v[c][r], S.part_k[c][r], bv, bk)) {
          bv = S.part_v[c][r];
          bk = S.part_k[c][r];
        }
      // row r -> the r-th live stream
      int i = 0;
      for (int seen = -1; i < ns; ++i)
        if (S.live[i] && ++seen == r) break;
      if (bk != 0) {
        const int32_t len = S.len[i];
        tokens[frame_splits[s0 + i] + len] = bk;
        S.len[i] = len + 1;
        S.ctx[i] = (S.ctx[i] % m.V) * m.V + bk;
      }
    }
    cluster.sync();  // contexts advanced
    if (rank != 0 && threadIdx.x < ns) S.ctx[threadIdx.x] = S0.ctx[threadIdx.x];
    __syncthreads();
  }
  if (rank == 0 && threadIdx.x < ns) lengths[s0 + threadIdx.x] = S.len[threadIdx.x];
  if (rank == 0 && threadIdx.x == 0) {
    unsigned long long sf = 0;
    for (int i = 0; i < ns; ++i) sf += frame_splits[s0 + i + 1] - frame_splits[s0 + i];
    atomicAdd(&counters[0], sf);
    atomicAdd(&counters[1], rows_total);
  }
  cluster.sync();  // no CTA leaves while others may still read its shared memory
}

}  // namespace

bool greedy_cluster_fits(const DeviceModel& d, int32_t B) {
  return B > 0 && B <= 18 * kClRows && d.Vp % kCl == 0 &&
         (static_cast<size_t>(d.J) * (d.Vp / kCl + kClRows)) * 4 + sizeof(ClSmem) <= 200 * 1024;
}

cudaError_t launch_decode_greedy_cluster(const DecodeArgs& a, cudaStream_t s) {
  const ModelView m = view_of(*a.m);
  // one stream per cluster up to 18 clusters (144 SMs), then up to 8 each
  const int nclusters = std::max((a.B + kClRows - 1) / kClRows, std::min(18, a.B));
  const int G = (a.B + nclusters - 1) / nclusters;
  const size_t smem = (static_cast<size_t>(m.J) * (m.Vp / kCl + kClRows)) * 4 + sizeof(ClSmem);
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
