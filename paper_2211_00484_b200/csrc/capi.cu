// C ABI of librnntg.so (include/rnntg.h): argument validation mirroring the
// reference's checks, device model construction, and the decode drivers.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <charconv>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

namespace rnntg {

static thread_local std::string g_error;
void set_error(const std::string& msg) { g_error = msg; }

}  // namespace rnntg

using rnntg::Scratch;
using rnntg::set_error;

struct rnntg_model_s {
  int device = 0;
  rnntg::DeviceModel d;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int num_sms = 1;
  int joiner_mode = RNNTG_JOINER_EXACT;
  // Time-sliced host-frame path for the beam kernel (copy + K1 of slice k+1
  // under the decode of slice k).  RNNTG_SLICED: 1 = host frames of uniform
  // length (default), 0 = never.
  // RNNTG_SLICE_FIRST / RNNTG_SLICE_MAX: first slice length (frames) and
  // the cap its doubling grows to.
  int sliced = 1;
  int32_t slice_first = 8, slice_max = 512;
  // RNNTG_SLICE_OVERLAP=1: K1 of slice k+1 on a second stream (fills the
  // decode tail of slice k) instead of in line on the compute stream.
  int slice_overlap = 1;
  int slice_throttle = 1;  // RNNTG_SLICE_THROTTLE=n: K1 k waits for decode k-1-n (0: no wait)
  cudaStream_t kstream = nullptr;
  std::vector<cudaEvent_t> k1_ev;  // one per slice: its pe rows are written
  Scratch hstate;                     // per-stream hypothesis sets between slices
  std::vector<cudaEvent_t> slice_ev;  // one per slice: its frames have landed
  Scratch pool;           // beam S > 1: sequence node pool
  // Small-batch greedy on thread-block clusters (cluster.cu);
  // RNNTG_GREEDY_CLUSTER=0 disables.
  bool greedy_cluster = true;
  // Small-batch beam search on thread-block clusters (decode.cu);
  // RNNTG_BEAM_CLUSTER=0 disables.
  bool beam_cluster = true;
  int32_t slot_mult = 1;  // token slots per frame of the current call (greedy S > 1)
  Scratch enc, pe, splits, tok, len, score, bp, counters, ctx, out_tok, out_splits, logits;
  Scratch finfo, nodebest, lattice, flag, feat, hid, fenc;
  Scratch nodectx, ladd_u, ladd_tot, ladd_narc, ladd_paths, ladd_cells, ladd_pos;  // log-add best sequences
  int32_t last_fsa_K = 0;
  // FSA step API (rnntg_fsa_stream_*): the open decode's graph, parameters,
  // frame splits, per-stream device state, and the rows of the last
  // rnntg_fsa_stream_contexts (host)
  rnntg_graph_t step_graph = nullptr;
  rnntg_fsa_params step_params{};
  std::vector<int32_t> step_fs, step_rows, step_nact;
  bool step_open = false, step_have_rows = false;
  Scratch step_state, step_P, step_rsplits;
  uint64_t ladd_seed = 0;
  int64_t ladd_n = 0, ladd_cell_cap = 4096;
  int64_t lat_cap_hint = 0;
  cudaStream_t cstream[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t done[4] = {nullptr, nullptr, nullptr, nullptr};
  bool pipelined = false;
  std::vector<int32_t> last_fsa_fs;  // frame splits of the last FSA call (lattice export)
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  rnntg_stats stats{};
  std::mutex mu;
  std::vector<void*> owned;  // device weight buffers
  std::vector<rnntg_graph_t> graphs;  // live graphs bound to this model (detached on destroy)
};

struct rnntg_graph_s {
  rnntg_model_t model = nullptr;
  int32_t num_states = 0, num_arcs = 0;
  int32_t max_out = 0;        // largest out-degree (step API lattice sizing)
  int32_t* splits = nullptr;  // device [S+1]
  void* arcs = nullptr;       // device 16-byte records {dst, label, weight}
  double* maxw = nullptr;     // device [S]: max outgoing arc weight per state
};

namespace {

int32_t round_up(int32_t x, int32_t m) { return (x + m - 1) / m * m; }

// NVTX ranges around every C-ABI decode call and its phases (SURVEY.md §5
// tracing): visible in Nsight Systems / ncu --nvtx without any code change.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

rnntg_status invalid(const std::string& msg) {
  set_error(msg);
  return RNNTG_INVALID_ARGUMENT;
}

template <typename T>
rnntg_status upload(rnntg_model_t h, T** dst, const std::vector<T>& src) {
  RNNTG_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(dst), sizeof(T) * std::max<size_t>(1, src.size())));
  h->owned.push_back(*dst);
  RNNTG_CUDA_TRY(cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice));
  return RNNTG_OK;
}

// k-major transpose with zero-padded columns: out[k][n] = w[n][k].
std::vector<float> transpose_pad(const float* w, int32_t N, int32_t K, int32_t ldo) {
  std::vector<float> out(static_cast<size_t>(K) * ldo, 0.0f);
  for (int32_t n = 0; n < N; ++n)
    for (int32_t k = 0; k < K; ++k) out[static_cast<size_t>(k) * ldo + n] = w[static_cast<size_t>(n) * K + k];
  return out;
}

// Validates the frame layout (one Mat per stream in the reference).
rnntg_status check_frames(const float* enc, const int32_t* fs, int32_t B) {
  if (B < 0) return invalid("batch size must be >= 0");
  if (B > 0 && fs == nullptr) return invalid("frame_splits is null");
  if (B > 0 && fs[0] != 0) return invalid("frame_splits[0] must be 0");
  for (int32_t i = 0; i < B; ++i)
    if (fs[i + 1] < fs[i]) return invalid("frame_splits must be non-decreasing");
  if (B > 0 && fs[B] > 0 && enc == nullptr) return invalid("enc is null");
  return RNNTG_OK;
}

rnntg_status encoder_impl(rnntg_model_t h, const float* feats, const int32_t* fs, int32_t B, int32_t mem,
                          float* enc_out) {
  const int64_t total = B > 0 ? fs[B] : 0;
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  const int32_t D = h->d.D, F = h->d.F, Dp = round_up(D, 128);
  const float* x = feats;
  float* y = enc_out;
  // HOST: host in, host out; DEVICE: device in and out; HOST_FEATURES
  // (internal, frames_from): host features in, device frames out.
  if (mem != RNNTG_MEM_DEVICE) {
    RNNTG_CUDA_TRY(h->feat.ensure(sizeof(float) * total * F));
    RNNTG_CUDA_TRY(cudaMemcpyAsync(h->feat.ptr, feats, sizeof(float) * total * F,
                                   cudaMemcpyHostToDevice, h->stream));
    x = h->feat.as<float>();
  }
  if (mem == RNNTG_MEM_HOST) {
    RNNTG_CUDA_TRY(h->enc.ensure(sizeof(float) * total * D));
    y = h->enc.as<float>();
  }
  RNNTG_CUDA_TRY(h->hid.ensure(sizeof(float) * total * D));
  // encoder_forward (model.hpp:224-238): two affine + tanh layers per frame.
  RNNTG_CUDA_TRY(rnntg::launch_gemm_exact(x, F, h->d.enc_w1t, Dp, h->d.enc_b1, h->hid.as<float>(), D,
                                          total, D, F, true, nullptr, 0, 0, h->stream));
  RNNTG_CUDA_TRY(rnntg::launch_gemm_exact(h->hid.as<float>(), D, h->d.enc_w2t, Dp, h->d.enc_b2, y, D,
                                          total, D, D, true, nullptr, 0, 0, h->stream));
  if (mem == RNNTG_MEM_HOST)
    RNNTG_CUDA_TRY(cudaMemcpyAsync(enc_out, y, sizeof(float) * total * D, cudaMemcpyDeviceToHost, h->stream));
  RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return RNNTG_OK;
}

bool mem_ok(int32_t mem) {
  return mem == RNNTG_MEM_HOST || mem == RNNTG_MEM_DEVICE || mem == RNNTG_MEM_HOST_FEATURES;
}

// RNNTG_MEM_HOST_FEATURES (the reference's own input, model.hpp:224-238):
// the GPU encoder turns the host features into device-resident frames
// (h->fenc); the search then runs on device frames and returns host
// results.  On return `enc` / `mem` describe the frames, `out_mem` the
// outputs.  Caller holds h->mu.
rnntg_status frames_from(rnntg_model_t h, const float*& enc, const int32_t* fs, int32_t B, int32_t& mem,
                         int32_t& out_mem) {
  out_mem = mem;
  if (mem != RNNTG_MEM_HOST_FEATURES) return RNNTG_OK;
  if (h->d.F == 0) return invalid("no encoder weights (rnntg_model_set_encoder)");
  const int64_t total = B > 0 ? fs[B] : 0;
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  RNNTG_CUDA_TRY(h->fenc.ensure(sizeof(float) * std::max<int64_t>(1, total) * h->d.D));
  if (total > 0) {
    rnntg_status st = encoder_impl(h, enc, fs, B, RNNTG_MEM_HOST_FEATURES, h->fenc.as<float>());
    if (st) return st;
  }
  enc = h->fenc.as<float>();
  mem = RNNTG_MEM_DEVICE;
  out_mem = RNNTG_MEM_HOST;
  return RNNTG_OK;
}

// Common front half of a decode call: buffers, splits, counters.
rnntg_status prepare(rnntg_model_t h, const int32_t* fs, int32_t B, int32_t mem) {
  Nvtx nvtx_range("rnntg: prepare (buffers, splits)");
  const int64_t total = B > 0 ? fs[B] : 0;
  const int32_t D = h->d.D, J = h->d.J;
  RNNTG_CUDA_TRY(h->splits.ensure(sizeof(int32_t) * (B + 1)));
  RNNTG_CUDA_TRY(cudaMemcpyAsync(h->splits.ptr, fs, sizeof(int32_t) * (B + 1),
                                 cudaMemcpyHostToDevice, h->stream));
  if (mem == RNNTG_MEM_HOST)
    RNNTG_CUDA_TRY(h->enc.ensure(sizeof(float) * std::max<int64_t>(1, total) * D));
  RNNTG_CUDA_TRY(h->pe.ensure(sizeof(float) * std::max<int64_t>(1, total) * J));
  RNNTG_CUDA_TRY(h->tok.ensure(sizeof(int32_t) * std::max<int64_t>(1, total * h->slot_mult)));
  RNNTG_CUDA_TRY(h->len.ensure(sizeof(int32_t) * std::max(1, B)));
  RNNTG_CUDA_TRY(h->score.ensure(sizeof(double) * std::max(1, B)));
  RNNTG_CUDA_TRY(h->counters.ensure(sizeof(unsigned long long) * 16));
  RNNTG_CUDA_TRY(cudaMemsetAsync(h->counters.ptr, 0, sizeof(unsigned long long) * 16, h->stream));
  return RNNTG_OK;
}

// Frames of uniform length T, decoded in time slices: slice k = frames
// [cut_k, cut_{k+1}) of every stream (lengths slice_first, doubling up to
// slice_max).  Host frames: a copy stream moves each slice with one pitched
// cudaMemcpy2DAsync and records the slice's event (device frames: the events
// are recorded at once).  K1 of the slice (row groups) runs on a side stream
// once its frames have landed — so it fills the SMs the previous slice's
// decode is draining — and the compute stream decodes the slice after it
// (beam kernel resuming from the hypothesis sets the previous slice stored).
// Only the first (short) slice's copy is exposed; K1 and decode keep the
// unfused kernels' machine code.
template <typename Launch>
rnntg_status run_sliced(rnntg_model_t h, const float* enc, const int32_t* fs, int32_t B, int32_t mem,
                        int64_t* launches, Launch&& launch) {
  const int32_t D = h->d.D, J = h->d.J, T = fs[1] - fs[0];
  // RNNTG_MEM_HOST_FEATURES: the slices carry acoustic features; the two
  // encoder layers of a slice run (row groups) in front of its K1
  const bool feat = mem == RNNTG_MEM_HOST_FEATURES;
  const int32_t F = h->d.F, Dp = round_up(D, 128);
  const int64_t total = static_cast<int64_t>(B) * T;
  if (feat) {
    RNNTG_CUDA_TRY(h->feat.ensure(sizeof(float) * std::max<int64_t>(1, total) * F));
    RNNTG_CUDA_TRY(h->hid.ensure(sizeof(float) * std::max<int64_t>(1, total) * D));
    RNNTG_CUDA_TRY(h->fenc.ensure(sizeof(float) * std::max<int64_t>(1, total) * D));
  }
  std::vector<int32_t> cut{0};
  for (int32_t len = h->slice_first; cut.back() < T; len = std::min(2 * len, std::max(h->slice_first, h->slice_max)))
    cut.push_back(std::min(T, cut.back() + len));
  const int nsl = static_cast<int>(cut.size()) - 1;
  RNNTG_CUDA_TRY(h->hstate.ensure(rnntg::beam_state_bytes() * static_cast<size_t>(B)));
  while (static_cast<int>(h->slice_ev.size()) < nsl) {
    cudaEvent_t e;
    RNNTG_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->slice_ev.push_back(e);
  }
  if (!h->cstream[0]) RNNTG_CUDA_TRY(cudaStreamCreateWithFlags(&h->cstream[0], cudaStreamNonBlocking));
  cudaStream_t cs = h->cstream[0];
  RNNTG_CUDA_TRY(cudaEventRecord(h->ev[0], h->stream));
  RNNTG_CUDA_TRY(cudaStreamWaitEvent(cs, h->ev[0], 0));  // the previous call is done with h->enc
  const size_t pitch = sizeof(float) * static_cast<size_t>(T) * D;
  const float* d_enc = feat ? h->fenc.as<float>() : mem == RNNTG_MEM_HOST ? h->enc.as<float>() : enc;
  for (int k = 0; k < nsl; ++k) {
    const int32_t f0 = cut[k], nf = cut[k + 1] - cut[k];
    if (feat) {
      const size_t fp = sizeof(float) * static_cast<size_t>(T) * F;
      RNNTG_CUDA_TRY(cudaMemcpy2DAsync(h->feat.as<float>() + static_cast<int64_t>(f0) * F, fp,
                                       enc + static_cast<int64_t>(f0) * F, fp, sizeof(float) * static_cast<size_t>(nf) * F,
                                       B, cudaMemcpyHostToDevice, cs));
      RNNTG_CUDA_TRY(cudaEventRecord(h->slice_ev[k], cs));
      continue;
    }
    if (mem != RNNTG_MEM_HOST) {  // frames already resident: the slice is ready now
      RNNTG_CUDA_TRY(cudaEventRecord(h->slice_ev[k], cs));
      continue;
    }
    RNNTG_CUDA_TRY(cudaMemcpy2DAsync(h->enc.as<float>() + static_cast<int64_t>(f0) * D, pitch, enc + static_cast<int64_t>(f0) * D,
                                     pitch, sizeof(float) * static_cast<size_t>(nf) * D, B,
                                     cudaMemcpyHostToDevice, cs));
    RNNTG_CUDA_TRY(cudaEventRecord(h->slice_ev[k], cs));
  }
  RNNTG_CUDA_TRY(cudaEventRecord(h->ev[1], h->stream));
  cudaStream_t ks = h->stream;
  if (h->slice_overlap) {
    if (!h->kstream) RNNTG_CUDA_TRY(cudaStreamCreateWithFlags(&h->kstream, cudaStreamNonBlocking));
    ks = h->kstream;
    while (static_cast<int>(h->k1_ev.size()) < 2 * nsl) {  // [k]: K1 k done; [nsl + k]: decode k done
      cudaEvent_t e;
      RNNTG_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->k1_ev.push_back(e);
    }
    RNNTG_CUDA_TRY(cudaStreamWaitEvent(ks, h->ev[1], 0));  // pe buffer free
  }
  for (int k = 0; k < nsl; ++k) {
    const int32_t f0 = cut[k], nf = cut[k + 1] - cut[k];
    RNNTG_CUDA_TRY(cudaStreamWaitEvent(ks, h->slice_ev[k], 0));
    // K1 of slice k is issued once decode k-2 is done, i.e. while decode k-1
    // runs: its CTAs take the SMs that decode drains at its tail instead of
    // delaying decode k-1's start.
    if (ks != h->stream && h->slice_throttle > 0 && k >= 1 + h->slice_throttle)
      RNNTG_CUDA_TRY(cudaStreamWaitEvent(ks, h->k1_ev[nsl + k - 1 - h->slice_throttle], 0));
    if (feat) {  // encoder_forward (model.hpp:224-238) of the slice: two affine + tanh layers
      RNNTG_CUDA_TRY(rnntg::launch_gemm_exact_grouped(
          h->feat.as<float>() + static_cast<int64_t>(f0) * F, F, h->d.enc_w1t, Dp, h->d.enc_b1,
          h->hid.as<float>() + static_cast<int64_t>(f0) * D, D, static_cast<int64_t>(B) * nf, D, F, true, nullptr, 0, 0,
          nf, T, ks));
      RNNTG_CUDA_TRY(rnntg::launch_gemm_exact_grouped(
          h->hid.as<float>() + static_cast<int64_t>(f0) * D, D, h->d.enc_w2t, Dp, h->d.enc_b2,
          h->fenc.as<float>() + static_cast<int64_t>(f0) * D, D, static_cast<int64_t>(B) * nf, D, D, true, nullptr, 0, 0,
          nf, T, ks));
      *launches += 2;
    }
    RNNTG_CUDA_TRY(rnntg::launch_gemm_exact_grouped(d_enc + static_cast<int64_t>(f0) * D, D, h->d.j_wet, h->d.Jp,
                                                    nullptr, h->pe.as<float>() + static_cast<int64_t>(f0) * J, J,
                                                    static_cast<int64_t>(B) * nf, J, D, false, nullptr, 0, 0, nf,
                                                    T, ks));
    if (ks != h->stream) {
      RNNTG_CUDA_TRY(cudaEventRecord(h->k1_ev[k], ks));
      RNNTG_CUDA_TRY(cudaStreamWaitEvent(h->stream, h->k1_ev[k], 0));
    }
    RNNTG_CUDA_TRY(launch(cut[k], cut[k + 1], h->stream));
    if (ks != h->stream) RNNTG_CUDA_TRY(cudaEventRecord(h->k1_ev[nsl + k], h->stream));
    *launches += 2;
  }
  h->pipelined = true;  // decode overlaps the copies: the stats report the whole call
  return RNNTG_OK;
}

// Runs frames -> pe -> decode.  Device-resident frames: one pe GEMM and one
// decode launch on the handle's stream.  Host frames: the batch is cut into
// up to kChunks stream ranges (multiples of the CTA stream group G); chunk c
// is copied, projected and decoded on its own CUDA stream, so the H2D copy of
// chunk c+1 overlaps the decode of chunk c and the decode kernels of
// different chunks share the SMs.  launch(b0, b1, stream) issues the decode
// kernel for streams [b0, b1).
template <typename Launch>
rnntg_status run_pipeline(rnntg_model_t h, const float* enc, const int32_t* fs, int32_t B,
                          int32_t mem, int32_t G, int64_t* launches, Launch&& launch) {
  constexpr int kChunks = 4;
  const int32_t D = h->d.D, J = h->d.J;
  const float* d_enc = mem == RNNTG_MEM_HOST ? h->enc.as<float>() : enc;
  int nch = 1;
  if (mem == RNNTG_MEM_HOST && B >= 2 * G) nch = std::min(kChunks, B / G);
  std::vector<int32_t> cut(nch + 1, 0);
  for (int c = 1; c < nch; ++c) cut[c] = static_cast<int32_t>((static_cast<int64_t>(B) / G * c / nch) * G);
  cut[nch] = B;
  RNNTG_CUDA_TRY(cudaEventRecord(h->ev[0], h->stream));
  for (int c = 0; c < nch; ++c) {
    const int32_t b0 = cut[c], b1 = cut[c + 1];
    if (b1 <= b0) continue;
    cudaStream_t cs = h->stream;
    if (nch > 1) {
      if (!h->cstream[c]) RNNTG_CUDA_TRY(cudaStreamCreateWithFlags(&h->cstream[c], cudaStreamNonBlocking));
      cs = h->cstream[c];
      RNNTG_CUDA_TRY(cudaStreamWaitEvent(cs, h->ev[0], 0));
    }
    const int64_t r0 = fs[b0], rows = fs[b1] - fs[b0];
    if (rows > 0) {
      if (mem == RNNTG_MEM_HOST)
        RNNTG_CUDA_TRY(cudaMemcpyAsync(h->enc.as<float>() + r0 * D, enc + r0 * D,
                                       sizeof(float) * rows * D, cudaMemcpyHostToDevice, cs));
      RNNTG_CUDA_TRY(rnntg::launch_gemm_exact(d_enc + r0 * D, D, h->d.j_wet, h->d.Jp, nullptr,
                                              h->pe.as<float>() + r0 * J, J, rows, J, D, false,
                                              nullptr, 0, 0, cs));
      ++*launches;
    }
    if (nch == 1) RNNTG_CUDA_TRY(cudaEventRecord(h->ev[1], h->stream));
    RNNTG_CUDA_TRY(launch(b0, b1, cs));
    ++*launches;
    if (nch > 1) {
      if (!h->done[c]) RNNTG_CUDA_TRY(cudaEventCreateWithFlags(&h->done[c], cudaEventDisableTiming));
      RNNTG_CUDA_TRY(cudaEventRecord(h->done[c], cs));
      RNNTG_CUDA_TRY(cudaStreamWaitEvent(h->stream, h->done[c], 0));
    }
  }
  if (nch > 1) RNNTG_CUDA_TRY(cudaEventRecord(h->ev[1], h->stream));
  h->pipelined = nch > 1;
  return RNNTG_OK;
}

__global__ void compact_tokens_kernel(const int32_t* __restrict__ slot_tokens,
                                      const int32_t* __restrict__ fs,
                                      const int32_t* __restrict__ out_splits,
                                      int32_t B, int32_t mult, int32_t* __restrict__ out) {
  const int s = blockIdx.x;
  if (s >= B) return;
  const int32_t n = out_splits[s + 1] - out_splits[s];
  const int64_t base = static_cast<int64_t>(mult) * fs[s];
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[out_splits[s] + i] = slot_tokens[base + i];
}

// Common back half: lengths -> out_splits, tokens compacted to the ragged
// layout, scores, stats.
rnntg_status finish(rnntg_model_t h, const int32_t* fs, int32_t B, int32_t mem,
                    int32_t* out_splits, int32_t* out_tokens, double* out_scores,
                    int64_t launches) {
  Nvtx nvtx_range("rnntg: results (compact + read back)");
  RNNTG_CUDA_TRY(cudaEventRecord(h->ev[2], h->stream));
  const int64_t total = B > 0 ? static_cast<int64_t>(fs[B]) * h->slot_mult : 0;
  std::vector<int32_t> lens(std::max(1, B));
  if (B > 0)
    RNNTG_CUDA_TRY(cudaMemcpyAsync(lens.data(), h->len.ptr, sizeof(int32_t) * B,
                                   cudaMemcpyDeviceToHost, h->stream));
  unsigned long long cnt[16];
  RNNTG_CUDA_TRY(cudaMemcpyAsync(cnt, h->counters.ptr, sizeof(cnt), cudaMemcpyDeviceToHost, h->stream));
  RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
  out_splits[0] = 0;
  for (int32_t i = 0; i < B; ++i) out_splits[i + 1] = out_splits[i] + lens[i];
  if (mem == RNNTG_MEM_HOST) {
    if (total > 0) {
      // Compact on the device, then read back only the hypothesis tokens
      // (~0.05 per frame here), not every per-frame token slot.
      const int64_t ntok = out_splits[B];
      RNNTG_CUDA_TRY(h->out_splits.ensure(sizeof(int32_t) * (B + 1)));
      RNNTG_CUDA_TRY(h->out_tok.ensure(sizeof(int32_t) * std::max<int64_t>(1, ntok)));
      RNNTG_CUDA_TRY(cudaMemcpyAsync(h->out_splits.ptr, out_splits, sizeof(int32_t) * (B + 1),
                                     cudaMemcpyHostToDevice, h->stream));
      compact_tokens_kernel<<<B, 128, 0, h->stream>>>(h->tok.as<int32_t>(), h->splits.as<int32_t>(),
                                                      h->out_splits.as<int32_t>(), B, h->slot_mult,
                                                      h->out_tok.as<int32_t>());
      RNNTG_CUDA_TRY(cudaGetLastError());
      ++launches;
      if (ntok > 0)
        RNNTG_CUDA_TRY(cudaMemcpyAsync(out_tokens, h->out_tok.ptr, sizeof(int32_t) * ntok,
                                       cudaMemcpyDeviceToHost, h->stream));
      if (out_scores)
        RNNTG_CUDA_TRY(cudaMemcpyAsync(out_scores, h->score.ptr, sizeof(double) * B,
                                       cudaMemcpyDeviceToHost, h->stream));
      RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
    } else if (out_scores && B > 0) {
      RNNTG_CUDA_TRY(cudaMemcpy(out_scores, h->score.ptr, sizeof(double) * B, cudaMemcpyDeviceToHost));
    }
  } else {
    RNNTG_CUDA_TRY(h->out_splits.ensure(sizeof(int32_t) * (B + 1)));
    RNNTG_CUDA_TRY(cudaMemcpyAsync(h->out_splits.ptr, out_splits, sizeof(int32_t) * (B + 1),
                                   cudaMemcpyHostToDevice, h->stream));
    if (B > 0 && total > 0) {
      compact_tokens_kernel<<<B, 128, 0, h->stream>>>(h->tok.as<int32_t>(), h->splits.as<int32_t>(),
                                                      h->out_splits.as<int32_t>(), B, h->slot_mult,
                                                      out_tokens);
      RNNTG_CUDA_TRY(cudaGetLastError());
      ++launches;
    }
    if (out_scores && B > 0)
      RNNTG_CUDA_TRY(cudaMemcpyAsync(out_scores, h->score.ptr, sizeof(double) * B,
                                     cudaMemcpyDeviceToDevice, h->stream));
    RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  float ms_all = 0, ms_dec = 0;
  cudaEventElapsedTime(&ms_all, h->ev[0], h->ev[2]);
  if (h->pipelined)  // decode overlaps the copies; report the whole call
    ms_dec = ms_all;
  else
    cudaEventElapsedTime(&ms_dec, h->ev[1], h->ev[2]);
  h->stats.stream_frames = static_cast<int64_t>(cnt[0]);
  h->stats.joiner_rows = static_cast<int64_t>(cnt[1]);
  h->stats.arcs_expanded = static_cast<int64_t>(cnt[2]);
  h->stats.lattice_arcs = static_cast<int64_t>(cnt[3]);
  h->stats.tie_breaks = static_cast<int64_t>(cnt[4]);
  h->stats.kernel_launches = launches;
  for (int i = 0; i < 4; ++i) h->stats.phase_cycles[i] = static_cast<int64_t>(cnt[8 + i]);
  h->stats.joiner_rows_computed = static_cast<int64_t>(cnt[5]);
  h->stats.gather_cycles = static_cast<int64_t>(cnt[6]);
  h->stats.capped_frames = h->slot_mult > 1 ? static_cast<int64_t>(cnt[13]) : 0;
  h->stats.gemm_wait_cycles = static_cast<int64_t>(cnt[7]);
  h->stats.gpu_ms = ms_all;
  h->stats.decode_ms = ms_dec;
  return RNNTG_OK;
}

}  // namespace

namespace {
// Host in, host out through temporary device buffers (debug entry points).
template <typename In, typename Out, typename F>
rnntg_status debug_roundtrip(int32_t device, const In* in, size_t n_in, Out* out, size_t n_out, F launch) {
  RNNTG_CUDA_TRY(cudaSetDevice(device));
  In* di = nullptr;
  Out* dout = nullptr;
  cudaError_t e = cudaMalloc(&di, sizeof(In) * std::max<size_t>(1, n_in));
  if (e == cudaSuccess) e = cudaMalloc(&dout, sizeof(Out) * std::max<size_t>(1, n_out));
  if (e == cudaSuccess) e = cudaMemcpy(di, in, sizeof(In) * n_in, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch(di, dout);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, sizeof(Out) * n_out, cudaMemcpyDeviceToHost);
  cudaFree(di);
  cudaFree(dout);
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return RNNTG_CUDA_ERROR;
  }
  return RNNTG_OK;
}
}  // namespace

extern "C" {

const char* rnntg_last_error(void) { return rnntg::g_error.c_str(); }
const char* rnntg_version(void) { return "rnntg 0.1 (sm_100a)"; }

rnntg_status rnntg_model_create(const rnntg_model_desc* desc, int32_t device,
                                rnntg_model_t* out) {
  Nvtx nvtx_range("rnntg_model_create");
  if (!desc || !out) return invalid("null argument");
  *out = nullptr;
  // check_config (model.hpp:174-182).
  if (desc->vocab_size < 2) return invalid("vocab_size must be >= 2 (blank plus one token)");
  if (desc->context_size != 2) return invalid("context_size must be 2");
  if (desc->enc_dim < 1 || desc->emb_dim < 1 || desc->joiner_dim < 1)
    return invalid("model dims must be >= 1");
  if (desc->joiner_dim > rnntg::kMaxJoiner) return invalid("joiner_dim too large");
  if (desc->vocab_size > rnntg::kMaxVocab) {
    set_error("vocab_size > 512 is beyond this build's joiner row cap");
    return RNNTG_UNSUPPORTED;
  }
  const float* ptrs[] = {desc->emb, desc->ctx_w, desc->ctx_b, desc->j_we,
                         desc->j_wd, desc->j_b, desc->out_w, desc->out_b};
  for (const float* p : ptrs)
    if (!p) return invalid("model weight pointer is null");
  const int32_t V = desc->vocab_size, D = desc->enc_dim, E = desc->emb_dim, J = desc->joiner_dim;
  const double table_bytes = static_cast<double>(V) * V * J * 4.0;
  if (table_bytes > 64.0 * (1ull << 30)) {
    set_error("decoder context table exceeds 64 GiB");
    return RNNTG_UNSUPPORTED;
  }

  RNNTG_CUDA_TRY(cudaSetDevice(device));
  auto* h = new rnntg_model_s();
  h->device = device;
  auto fail = [&](rnntg_status st) {
    rnntg_model_destroy(h);
    return st;
  };
  if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    set_error("cudaStreamCreate failed");
    delete h;
    return RNNTG_CUDA_ERROR;
  }
  h->stream = h->own_stream;
  for (auto& e : h->ev) cudaEventCreate(&e);
  h->num_sms = rnntg::decode_num_sms(device);
  if (const char* e = std::getenv("RNNTG_SLICED")) h->sliced = std::atoi(e);
  if (const char* e = std::getenv("RNNTG_SLICE_FIRST")) h->slice_first = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("RNNTG_SLICE_MAX")) h->slice_max = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("RNNTG_SLICE_OVERLAP")) h->slice_overlap = std::atoi(e);
  if (const char* e = std::getenv("RNNTG_SLICE_THROTTLE")) h->slice_throttle = std::atoi(e);
  if (const char* gc = std::getenv("RNNTG_GREEDY_CLUSTER")) h->greedy_cluster = std::atoi(gc) != 0;
  if (const char* bc = std::getenv("RNNTG_BEAM_CLUSTER")) h->beam_cluster = std::atoi(bc) != 0;
  rnntg::DeviceModel& d = h->d;
  d.V = V;
  d.D = D;
  d.E = E;
  d.J = J;
  d.Vp = round_up(V, 256);
  d.Ep = round_up(E, 128);
  d.Jp = round_up(J, 128);
  rnntg_status st;
  if ((st = upload(h, &d.emb, std::vector<float>(desc->emb, desc->emb + static_cast<size_t>(V) * E))) ||
      (st = upload(h, &d.ctx_wt, transpose_pad(desc->ctx_w, E, 2 * E, d.Ep))) ||
      (st = upload(h, &d.ctx_b, std::vector<float>(desc->ctx_b, desc->ctx_b + E))) ||
      (st = upload(h, &d.j_wet, transpose_pad(desc->j_we, J, D, d.Jp))) ||
      (st = upload(h, &d.j_wdt, transpose_pad(desc->j_wd, J, E, d.Jp))) ||
      (st = upload(h, &d.j_b, std::vector<float>(desc->j_b, desc->j_b + J))) ||
      (st = upload(h, &d.out_wt, transpose_pad(desc->out_w, V, J, d.Vp))))
    return fail(st);
  {
    std::vector<float> ob(d.Vp, 0.0f);
    std::copy(desc->out_b, desc->out_b + V, ob.begin());
    if ((st = upload(h, &d.out_b, ob))) return fail(st);
    if ((st = upload(h, &d.zeros, std::vector<float>(std::max(d.Vp, d.Jp), 0.0f)))) return fail(st);
  }
  if (J % 16 == 0) {
    // bf16 out_w for the tcgen05 variant, pre-arranged chunk by chunk (16
    // k-values per chunk) in the no-swizzle K-major UMMA core-matrix layout
    // so each chunk is one contiguous cp.async.bulk (decode_common.cuh).
    const int BK = 16;
    std::vector<uint16_t> wt(static_cast<size_t>(J) * d.Vp, 0);
    for (int32_t c = 0; c < J / BK; ++c)
      for (int32_t v = 0; v < d.Vp; ++v)
        for (int32_t kk = 0; kk < BK; ++kk) {
          const float x = v < V ? desc->out_w[static_cast<size_t>(v) * J + c * BK + kk] : 0.0f;
          uint32_t u;
          std::memcpy(&u, &x, 4);
          const uint32_t rnd = u + 0x7fffu + ((u >> 16) & 1u);  // round to nearest even
          const size_t off = static_cast<size_t>(c) * d.Vp * BK +
                             ((v >> 3) * (BK / 8) * 64 + (kk >> 3) * 64 + (v & 7) * 8 + (kk & 7));
          wt[off] = static_cast<uint16_t>(rnd >> 16);
        }
    if ((st = upload(h, &d.out_w_bf16, wt))) return fail(st);
  }
  // K0: the decoder-side joiner projection of every packed context,
  // pd[c] = j_wd . tanh(ctx_b + ctx_w . [emb[c/V]; emb[c%V]]), chunked.
  const int64_t C = static_cast<int64_t>(V) * V;
  if (cudaMalloc(reinterpret_cast<void**>(&d.pd_table), sizeof(float) * C * J) != cudaSuccess) {
    set_error("cannot allocate the decoder context table");
    return fail(RNNTG_CUDA_ERROR);
  }
  h->owned.push_back(d.pd_table);
  const int64_t chunk = 32768;
  float* dec = nullptr;
  if (cudaMalloc(reinterpret_cast<void**>(&dec), sizeof(float) * chunk * E) != cudaSuccess) {
    set_error("cannot allocate decoder scratch");
    return fail(RNNTG_CUDA_ERROR);
  }
  for (int64_t c0 = 0; c0 < C; c0 += chunk) {
    const int64_t n = std::min(chunk, C - c0);
    cudaError_t e = rnntg::launch_gemm_exact(nullptr, 0, d.ctx_wt, d.Ep, d.ctx_b, dec, E, n, E,
                                             2 * E, true, d.emb, V, c0, h->stream);
    if (e == cudaSuccess)
      e = rnntg::launch_gemm_exact(dec, E, d.j_wdt, d.Jp, nullptr, d.pd_table + c0 * J, J, n, J, E,
                                   false, nullptr, 0, 0, h->stream);
    if (e != cudaSuccess) {
      cudaFree(dec);
      set_error(std::string("decoder table: ") + cudaGetErrorString(e));
      return fail(RNNTG_CUDA_ERROR);
    }
  }
  cudaError_t e = cudaStreamSynchronize(h->stream);
  cudaFree(dec);
  if (e != cudaSuccess) {
    set_error(std::string("decoder table: ") + cudaGetErrorString(e));
    return fail(RNNTG_CUDA_ERROR);
  }
  *out = h;
  return RNNTG_OK;
}

rnntg_status rnntg_host_alloc(size_t bytes, void** out) {
  if (!out) return invalid("null argument");
  *out = nullptr;
  if (bytes == 0) return RNNTG_OK;
  if (cudaHostAlloc(out, bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    set_error("cudaHostAlloc failed");
    return RNNTG_CUDA_ERROR;
  }
  return RNNTG_OK;
}

rnntg_status rnntg_host_free(void* ptr) {
  if (ptr && cudaFreeHost(ptr) != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaFreeHost failed");
    return RNNTG_CUDA_ERROR;
  }
  return RNNTG_OK;
}

rnntg_status rnntg_model_destroy(rnntg_model_t h) {
  if (!h) return RNNTG_OK;
  {
    // graphs may outlive their model (destroyed later, in any order): they
    // are detached and refuse further searches
    std::lock_guard<std::mutex> lk(h->mu);
    for (rnntg_graph_t g : h->graphs) g->model = nullptr;
    h->graphs.clear();
  }
  cudaSetDevice(h->device);
  if (h->own_stream) cudaStreamSynchronize(h->own_stream);
  for (void* p : h->owned) cudaFree(p);
  for (Scratch* s : {&h->enc, &h->pe, &h->splits, &h->tok, &h->len, &h->score, &h->bp,
                     &h->counters, &h->ctx, &h->out_tok, &h->out_splits, &h->logits,
                     &h->finfo, &h->nodebest, &h->lattice, &h->flag, &h->feat, &h->hid,
                     &h->hstate, &h->pool, &h->fenc, &h->nodectx, &h->ladd_u, &h->ladd_tot,
                     &h->ladd_narc, &h->ladd_paths, &h->ladd_cells, &h->ladd_pos, &h->step_state, &h->step_P,
                     &h->step_rsplits})
    s->release();
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : h->slice_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : h->k1_ev) cudaEventDestroy(e);
  if (h->kstream) cudaStreamDestroy(h->kstream);
  for (int c = 0; c < 4; ++c) {
    if (h->cstream[c]) cudaStreamDestroy(h->cstream[c]);
    if (h->done[c]) cudaEventDestroy(h->done[c]);
  }
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
  return RNNTG_OK;
}

rnntg_status rnntg_set_stream(rnntg_model_t h, void* stream) {
  if (!h) return invalid("null model");
  std::lock_guard<std::mutex> lk(h->mu);
  h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own_stream;
  return RNNTG_OK;
}

rnntg_status rnntg_set_joiner_mode(rnntg_model_t h, int32_t mode) {
  if (!h) return invalid("null model");
  if (mode != RNNTG_JOINER_EXACT && mode != RNNTG_JOINER_BF16) return invalid("bad joiner mode");
  if (mode == RNNTG_JOINER_BF16 && !h->d.out_w_bf16) {
    set_error("bf16 tcgen05 joiner needs joiner_dim % 16 == 0");
    return RNNTG_UNSUPPORTED;
  }
  std::lock_guard<std::mutex> lk(h->mu);
  h->joiner_mode = mode;
  return RNNTG_OK;
}

rnntg_status rnntg_get_stats(rnntg_model_t h, rnntg_stats* out) {
  if (!h || !out) return invalid("null argument");
  *out = h->stats;
  return RNNTG_OK;
}

namespace {
// Greedy body shared by greedy_search_batch (cap 1) and greedy_search (cap
// = S, or 10 with the frames stopped by the cap counted when S is
// unlimited).  Caller holds h->mu and has validated the arguments.
rnntg_status greedy_impl(rnntg_model_t h, const float* enc, const int32_t* fs, int32_t B, int32_t cap,
                         bool count_capped, int32_t mem, int32_t* out_splits, int32_t* out_tokens) {
  int32_t out_mem = mem;
  rnntg_status st0 = frames_from(h, enc, fs, B, mem, out_mem);
  if (st0) return st0;
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  h->slot_mult = cap;
  rnntg_status st = prepare(h, fs, B, mem);
  if (st) {
    h->slot_mult = 1;
    return st;
  }
  int64_t launches = 0;
  if (B > 0) {
    const int G = std::min(32, std::max(1, (B + h->num_sms - 1) / h->num_sms));
    RNNTG_CUDA_TRY(cudaMemsetAsync(h->score.ptr, 0, sizeof(double) * B, h->stream));
    st = run_pipeline(h, enc, fs, B, mem, G, &launches, [&](int32_t b0, int32_t b1, cudaStream_t cs) {
      rnntg::DecodeArgs a{};
      a.m = &h->d;
      a.pe = h->pe.as<float>();
      a.frame_splits = h->splits.as<int32_t>() + b0;
      a.B = b1 - b0;
      a.streams_per_cta = G;
      a.tokens = h->tok.as<int32_t>();
      a.lengths = h->len.as<int32_t>() + b0;
      a.scores = h->score.as<double>() + b0;
      a.counters = h->counters.as<unsigned long long>();
      a.symbol_cap = cap;
      a.count_capped = count_capped ? 1 : 0;
      if (cap == 1 && h->greedy_cluster && rnntg::greedy_cluster_fits(h->d, b1 - b0))
        return rnntg::launch_decode_greedy_cluster(a, cs);
      return rnntg::launch_decode_greedy(a, cs);
    });
    if (st) {
      h->slot_mult = 1;
      return st;
    }
  }
  st = finish(h, fs, B, out_mem, out_splits, out_tokens, nullptr, launches);
  h->slot_mult = 1;
  return st;
}
}  // namespace

rnntg_status rnntg_greedy_search_batch(rnntg_model_t h, const float* enc,
                                       const int32_t* fs, int32_t B,
                                       int32_t max_symbols, int32_t mem,
                                       int32_t* out_splits, int32_t* out_tokens) {
  Nvtx nvtx_range("rnntg_greedy_search_batch");
  if (!h) return invalid("null model");
  // search.hpp:110-111.
  if (max_symbols != 1) return invalid("greedy_search_batch supports max_symbols = 1 only");
  if (!mem_ok(mem)) return invalid("bad mem kind");
  rnntg_status st = check_frames(enc, fs, B);
  if (st) return st;
  if (!out_splits) return invalid("out_splits is null");
  std::lock_guard<std::mutex> lk(h->mu);
  return greedy_impl(h, enc, fs, B, 1, false, mem, out_splits, out_tokens);
}

rnntg_status rnntg_greedy_search(rnntg_model_t h, const float* enc, const int32_t* fs, int32_t B,
                                 int32_t max_symbols, int32_t mem, int32_t* out_splits,
                                 int32_t* out_tokens, int64_t* capped_frames) {
  Nvtx nvtx_range("rnntg_greedy_search");
  if (!h) return invalid("null model");
  // search.hpp:80 and 31-34 (kNoSymbolLimit -> kMaxSymbolsPerFrameSafety = 10).
  if (max_symbols < 1) return invalid("max_symbols must be >= 1");
  if (!mem_ok(mem)) return invalid("bad mem kind");
  rnntg_status st = check_frames(enc, fs, B);
  if (st) return st;
  if (!out_splits) return invalid("out_splits is null");
  const bool unlimited = max_symbols == RNNTG_NO_SYMBOL_LIMIT;
  const int32_t cap = unlimited ? 10 : max_symbols;
  std::lock_guard<std::mutex> lk(h->mu);
  st = greedy_impl(h, enc, fs, B, cap, unlimited, mem, out_splits, out_tokens);
  if (!st && capped_frames) *capped_frames = h->stats.capped_frames;
  return st;
}

rnntg_status rnntg_beam_search_batch(rnntg_model_t h, const float* enc,
                                     const int32_t* fs, int32_t B,
                                     const rnntg_beam_params* p, int32_t mem,
                                     int32_t* out_splits, int32_t* out_tokens,
                                     double* out_scores) {
  Nvtx nvtx_range("rnntg_beam_search_batch");
  if (!h || !p) return invalid("null argument");
  // beam_search validation, search.hpp:210-212.
  if (p->max_symbols < 1) return invalid("max_symbols must be >= 1");
  if (p->beam_size < 1) return invalid("beam_size must be >= 1");
  if (p->beam_size > rnntg::kMaxBeam) {
    set_error("beam_size > 8 is beyond this build's per-stream hypothesis cap");
    return RNNTG_UNSUPPORTED;
  }
  if (p->merge_op != RNNTG_MERGE_MAX && p->merge_op != RNNTG_MERGE_LOG_ADD) return invalid("bad merge_op");
  if (!mem_ok(mem)) return invalid("bad mem kind");
  rnntg_status st = check_frames(enc, fs, B);
  if (st) return st;
  if (!out_splits) return invalid("out_splits is null");
  std::lock_guard<std::mutex> lk(h->mu);
  int32_t out_mem = mem;
  // Host features of a uniform batch that will be decoded in time slices:
  // the encoder runs per slice inside run_sliced (copies, encoder, K1 and
  // decode overlap) instead of all up front.
  bool feat_sliced = false;
  if (mem == RNNTG_MEM_HOST_FEATURES && B > 0 && p->max_symbols == 1 && h->joiner_mode == RNNTG_JOINER_EXACT &&
      h->sliced > 0 && h->d.F > 0 && fs[1] - fs[0] > h->slice_first) {
    bool uni = true;
    for (int32_t i = 1; i < B; ++i) uni = uni && fs[i + 1] - fs[i] == fs[1] - fs[0];
    feat_sliced = uni && !(h->beam_cluster && rnntg::beam_cluster_streams(h->d, B, p->beam_size, h->num_sms) > 0);
  }
  if (feat_sliced) {
    out_mem = RNNTG_MEM_HOST;
  } else if ((st = frames_from(h, enc, fs, B, mem, out_mem))) {
    return st;
  }
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  // S > 1 (search.hpp:228-235): up to `cap` sub-steps per frame, cap = 10
  // for kNoSymbolLimit (frames stopped by it counted in the stats).
  const bool unlimited = p->max_symbols == RNNTG_NO_SYMBOL_LIMIT;
  const int32_t cap = unlimited ? 10 : p->max_symbols;
  if (cap > 10) {
    set_error("beam search with 10 < max_symbols < unlimited is beyond this build's per-frame cap");
    return RNNTG_UNSUPPORTED;
  }
  h->slot_mult = cap;
  struct SlotReset {
    rnntg_model_t h;
    ~SlotReset() { h->slot_mult = 1; }
  } slot_reset{h};
  if ((st = prepare(h, fs, B, feat_sliced ? RNNTG_MEM_DEVICE : mem))) return st;
  int64_t launches = 0;
  if (B > 0 && cap > 1) {
    RNNTG_CUDA_TRY(h->pool.ensure(sizeof(int32_t) * 2 * (static_cast<int64_t>(fs[B]) * cap + B) * rnntg::kMaxBeam));
    const int gmax = std::max(1, 32 / p->beam_size);
    const int G = std::min(gmax, std::max(1, (B + h->num_sms - 1) / h->num_sms));
    st = run_pipeline(h, enc, fs, B, mem, G, &launches, [&](int32_t b0, int32_t b1, cudaStream_t cs) {
      rnntg::DecodeArgs a{};
      a.m = &h->d;
      a.pe = h->pe.as<float>();
      a.frame_splits = h->splits.as<int32_t>() + b0;
      a.B = b1 - b0;
      a.streams_per_cta = G;
      a.tokens = h->tok.as<int32_t>();
      a.lengths = h->len.as<int32_t>() + b0;
      a.scores = h->score.as<double>() + b0;
      a.counters = h->counters.as<unsigned long long>();
      a.beam_size = p->beam_size;
      a.merge_op = p->merge_op;
      a.length_norm = p->length_norm;
      a.max_total = p->max_total_symbols;
      a.symbol_cap = cap;
      a.count_capped = unlimited ? 1 : 0;
      a.node_pool = h->pool.as<int32_t>() + 2 * static_cast<int64_t>(b0);  // region base uses the global stream index
      return rnntg::launch_decode_beam(a, cs);
    });
    if (st) return st;
    return finish(h, fs, B, out_mem, out_splits, out_tokens, out_scores, launches);
  }
  if (B > 0) {
    const int64_t total = fs[B];
    RNNTG_CUDA_TRY(h->bp.ensure(sizeof(uint32_t) * (total + B) * rnntg::kMaxBeam));
    // Streams per CTA: enough to give every SM work, capped by the 32-row
    // joiner tile (and, for the warp-specialised kernel, 16 rows per half).
    const bool exact = h->joiner_mode == RNNTG_JOINER_EXACT;
    // Batches beyond one wave (num_sms * gmax streams) run in whole waves of
    // equal CTAs: G = ceil(B / (waves * num_sms)), not gmax with a ragged
    // last wave (B = 2048: 2 x 148 CTAs of 7 streams, not 148 + 108 of 8).
    const int gmax = std::max(1, exact ? 2 * (16 / p->beam_size) : 32 / p->beam_size);
    const int64_t waves = (static_cast<int64_t>(B) + static_cast<int64_t>(h->num_sms) * gmax - 1) /
                          (static_cast<int64_t>(h->num_sms) * gmax);
    const int G = std::min<int64_t>(gmax, std::max<int64_t>(1, (B + waves * h->num_sms - 1) / (waves * h->num_sms)));
    bool uniform = true;
    for (int32_t i = 1; i < B; ++i) uniform = uniform && fs[i + 1] - fs[i] == fs[1] - fs[0];
    auto args = [&](int32_t b0, int32_t b1) {
      rnntg::DecodeArgs a{};
      a.m = &h->d;
      a.pe = h->pe.as<float>();
      a.frame_splits = h->splits.as<int32_t>() + b0;
      a.B = b1 - b0;
      a.streams_per_cta = G;
      a.tokens = h->tok.as<int32_t>();
      a.lengths = h->len.as<int32_t>() + b0;
      a.scores = h->score.as<double>() + b0;
      a.counters = h->counters.as<unsigned long long>();
      a.beam_size = p->beam_size;
      a.merge_op = p->merge_op;
      a.length_norm = p->length_norm;
      a.max_total = p->max_total_symbols;
      // back-pointer rows are indexed (frame offset + stream index)
      a.backptr = h->bp.as<uint32_t>() + static_cast<int64_t>(b0) * rnntg::kMaxBeam;
      a.joiner_bf16 = h->joiner_mode == RNNTG_JOINER_BF16;
      return a;
    };
    // Small batches: the thread-block-cluster kernel (out_w column slices
    // resident in shared memory, decode.cu beam_cluster_kernel), one launch.
    const int Gc = exact && h->beam_cluster ? rnntg::beam_cluster_streams(h->d, B, p->beam_size, h->num_sms) : 0;
    if (Gc > 0) {
      st = run_pipeline(h, enc, fs, B, mem, B, &launches, [&](int32_t b0, int32_t b1, cudaStream_t cs) {
        rnntg::DecodeArgs a = args(b0, b1);
        a.streams_per_cta = Gc;  // streams per cluster
        return rnntg::launch_decode_beam_cluster(a, cs);
      });
      if (st) return st;
      return finish(h, fs, B, out_mem, out_splits, out_tokens, out_scores, launches);
    }
    const bool sliced = feat_sliced || (exact && uniform && fs[1] - fs[0] > h->slice_first &&
                                        ((mem == RNNTG_MEM_HOST && h->sliced > 0) ||
                                         (mem == RNNTG_MEM_DEVICE && h->sliced > 1)));
    if (sliced) {
      st = run_sliced(h, enc, fs, B, mem, &launches, [&](int32_t t0, int32_t t1, cudaStream_t cs) {
        rnntg::DecodeArgs a = args(0, B);
        a.t0 = t0;
        a.t1 = t1;
        a.hyps_state = h->hstate.ptr;
        return rnntg::launch_decode_beam(a, cs);
      });
      if (st) return st;
      return finish(h, fs, B, out_mem, out_splits, out_tokens, out_scores, launches);
    }
    st = run_pipeline(h, enc, fs, B, mem, G, &launches, [&](int32_t b0, int32_t b1, cudaStream_t cs) {
      rnntg::DecodeArgs a = args(b0, b1);
      return rnntg::launch_decode_beam(a, cs);
    });
    if (st) return st;
  }
  return finish(h, fs, B, out_mem, out_splits, out_tokens, out_scores, launches);
}

rnntg_status rnntg_graph_create(rnntg_model_t h, int32_t num_states,
                                const int32_t* arc_splits, int32_t num_arcs,
                                const int32_t* dst, const int32_t* label,
                                const double* weight, rnntg_graph_t* out) {
  Nvtx nvtx_range("rnntg_graph_create");
  if (!h || !out) return invalid("null argument");
  *out = nullptr;
  if (num_states < 1) return invalid("fsa must have at least one state");
  if (num_arcs < 0 || !arc_splits) return invalid("bad arc list");
  if (arc_splits[0] != 0 || arc_splits[num_states] != num_arcs)
    return invalid("arc_splits must start at 0 and end at num_arcs");
  int32_t max_out = 0;
  for (int32_t s = 0; s < num_states; ++s) {
    if (arc_splits[s + 1] < arc_splits[s]) return invalid("arc_splits must be non-decreasing");
    max_out = std::max(max_out, arc_splits[s + 1] - arc_splits[s]);
  }
  for (int32_t a = 0; a < num_arcs; ++a) {
    if (dst[a] < 0 || dst[a] >= num_states) return invalid("arc references state out of range");
    // init_streams, fsa_search.hpp:103-111.
    if (label[a] == 0) return invalid("decoding graph contains a blank/epsilon (label 0) arc");
    if (label[a] < 0 || label[a] >= h->d.V)
      return invalid("decoding graph label " + std::to_string(label[a]) + " outside model vocabulary");
    if (!std::isfinite(weight[a])) return invalid("arc score must be finite");
  }
  std::lock_guard<std::mutex> lk(h->mu);
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  auto* g = new rnntg_graph_s();  // bound to h once complete (error paths destroy it unbound)
  g->num_states = num_states;
  g->num_arcs = num_arcs;
  g->max_out = max_out;
  struct ArcRec {
    int32_t dst, label;
    double w;
  };
  std::vector<ArcRec> rec(std::max(1, num_arcs));
  for (int32_t a = 0; a < num_arcs; ++a) rec[a] = {dst[a], label[a], weight[a]};
  if (cudaMalloc(&g->arcs, sizeof(ArcRec) * rec.size()) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&g->splits), sizeof(int32_t) * (num_states + 1)) != cudaSuccess) {
    rnntg_graph_destroy(g);
    set_error("cannot allocate the device graph");
    return RNNTG_CUDA_ERROR;
  }
  cudaMemcpy(g->arcs, rec.data(), sizeof(ArcRec) * rec.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(g->splits, arc_splits, sizeof(int32_t) * (num_states + 1), cudaMemcpyHostToDevice);
  {
    std::vector<double> mw(num_states, -HUGE_VAL);
    for (int32_t s = 0; s < num_states; ++s)
      for (int32_t a = arc_splits[s]; a < arc_splits[s + 1]; ++a) mw[s] = std::max(mw[s], weight[a]);
    if (cudaMalloc(reinterpret_cast<void**>(&g->maxw), sizeof(double) * num_states) != cudaSuccess) {
      rnntg_graph_destroy(g);
      set_error("cannot allocate the device graph");
      return RNNTG_CUDA_ERROR;
    }
    cudaMemcpy(g->maxw, mw.data(), sizeof(double) * num_states, cudaMemcpyHostToDevice);
  }
  g->model = h;
  h->graphs.push_back(g);
  *out = g;
  return RNNTG_OK;
}

rnntg_status rnntg_graph_destroy(rnntg_graph_t g) {
  if (!g) return RNNTG_OK;
  if (g->model) {  // an open step decode over this graph ends with it
    std::lock_guard<std::mutex> lk(g->model->mu);
    if (g->model->step_graph == g) {
      g->model->step_open = false;
      g->model->step_graph = nullptr;
    }
    auto& gs = g->model->graphs;
    gs.erase(std::remove(gs.begin(), gs.end(), g), gs.end());
  }
  if (g->arcs) cudaFree(g->arcs);
  if (g->splits) cudaFree(g->splits);
  if (g->maxw) cudaFree(g->maxw);
  delete g;
  return RNNTG_OK;
}

rnntg_status rnntg_fsa_beam_search(rnntg_model_t h, const float* enc,
                                   const int32_t* fs, int32_t B,
                                   rnntg_graph_t graph,
                                   const rnntg_fsa_params* p, int32_t mem,
                                   int32_t* out_splits, int32_t* out_tokens,
                                   double* out_scores) {
  Nvtx nvtx_range("rnntg_fsa_beam_search");
  if (!h || !p || !graph) return invalid("null argument");
  if (graph->model != h) return invalid("graph belongs to another model handle");
  // check_fsa_search_params, fsa_search.hpp:83-90.
  if (!(p->beam >= 0.0)) return invalid("fsa search beam must be >= 0");
  if (p->max_states < 1) return invalid("max_states must be >= 1");
  if (p->max_contexts < 1) return invalid("max_contexts must be >= 1");
  if (!mem_ok(mem)) return invalid("bad mem kind");
  rnntg_status st = check_frames(enc, fs, B);
  if (st) return st;
  if (!out_splits) return invalid("out_splits is null");
  std::lock_guard<std::mutex> lk(h->mu);
  // The lattice buffers are overwritten below; until this call succeeds there
  // is no exportable lattice (rnntg_fsa_lattice).
  h->last_fsa_fs.clear();
  int32_t out_mem = mem;
  if ((st = frames_from(h, enc, fs, B, mem, out_mem))) return st;
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  if ((st = prepare(h, fs, B, mem))) return st;
  int64_t launches = 0;
  if (B > 0) {
    const int64_t total = fs[B];
    const int K = std::min(p->max_states, rnntg::kFsaMaxStates);
    const int rows = std::min(p->max_contexts, K);
    int G = 1;
    const int want = std::min({4, std::max(1, (B + h->num_sms - 1) / h->num_sms), std::max(1, 32 / rows)});
    while (G * 2 <= want) G *= 2;
    RNNTG_CUDA_TRY(h->finfo.ensure(sizeof(int32_t) * 4 * (total + B)));
    RNNTG_CUDA_TRY(h->nodebest.ensure(sizeof(double) * (total * K + B)));
    RNNTG_CUDA_TRY(h->nodectx.ensure(sizeof(int32_t) * (total * K + B)));
    RNNTG_CUDA_TRY(h->flag.ensure(16));
    // Lattice pool: sized so one decode suffices at the measured occupancy
    // (config 3: ~6.3, config 4: ~13 kept arcs per stream-frame against
    // max_states 8 / 64), i.e. 2K + 8 arcs per stream-frame, capped at 4 GiB
    // of 24-byte arcs; beyond that an overflow regrows it and decodes again.
    const int64_t want_cap = std::min<int64_t>(total * (2 * K + 8), (4ll << 30) / 24);
    int64_t cap = std::max<int64_t>({int64_t{1} << 20, h->lat_cap_hint, want_cap});
    const char* cap_knob = std::getenv("RNNTG_LAT_CAP");  // test knob: start from a small pool
    if (cap_knob) cap = std::max<int64_t>(1024, std::atoll(cap_knob));
    for (int attempt = 0;; ++attempt) {
      if (attempt == 0 && cap_knob) h->lattice.release();
      RNNTG_CUDA_TRY(h->lattice.ensure(static_cast<size_t>(cap) * 24));
      cap = static_cast<int64_t>(h->lattice.bytes / 24);
      RNNTG_CUDA_TRY(cudaMemsetAsync(h->flag.ptr, 0, 16, h->stream));
      RNNTG_CUDA_TRY(cudaMemsetAsync(h->counters.ptr, 0, sizeof(unsigned long long) * 16, h->stream));
      st = run_pipeline(h, enc, fs, B, mem, G, &launches, [&](int32_t b0, int32_t b1, cudaStream_t cs) {
        rnntg::DecodeArgs a{};
        a.m = &h->d;
        a.pe = h->pe.as<float>();
        a.frame_splits = h->splits.as<int32_t>() + b0;
        a.B = b1 - b0;
        a.streams_per_cta = G;
        a.tokens = h->tok.as<int32_t>();
        a.lengths = h->len.as<int32_t>() + b0;
        a.scores = h->score.as<double>() + b0;
        a.counters = h->counters.as<unsigned long long>();
        a.graph_arcs = graph->arcs;
        a.graph_splits = graph->splits;
        a.graph_maxw = graph->maxw;
        a.graph_states = graph->num_states;
        a.fsa_beam = p->beam;
        a.max_states = p->max_states;
        a.max_contexts = p->max_contexts;
        a.lattice = h->lattice.ptr;
        a.lattice_cap = cap;
        a.error_flag = h->flag.as<int32_t>();
        a.lattice_count = reinterpret_cast<unsigned long long*>(h->flag.as<char>() + 8);
        // per-(stream, frame) and per-node tables are indexed (frame offset + stream index)
        a.lat_frame_info = h->finfo.as<int32_t>() + 4 * static_cast<int64_t>(b0);
        a.node_best = h->nodebest.as<double>() + b0;
        a.node_ctx = h->nodectx.as<int32_t>() + b0;
        return rnntg::launch_decode_fsa(a, cs);
      });
      if (st) return st;
      int32_t flag = 0;
      unsigned long long used = 0;
      RNNTG_CUDA_TRY(cudaMemcpyAsync(&flag, h->flag.ptr, sizeof(flag), cudaMemcpyDeviceToHost, h->stream));
      RNNTG_CUDA_TRY(cudaMemcpyAsync(&used, h->flag.as<char>() + 8, sizeof(used), cudaMemcpyDeviceToHost, h->stream));
      RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
      if (flag == 1 && attempt < 4) {  // lattice pool overflow: grow and rerun
        cap = static_cast<int64_t>(used) * 2 + 1024;
        h->lat_cap_hint = cap;
        continue;
      }
      if (flag == 2) {
        set_error("more than 32 distinct contexts per CTA frame (max_contexts too large for this build)");
        return RNNTG_UNSUPPORTED;
      }
      if (flag == 3) {
        set_error("candidate hash overflow (too many exact-score duplicates near the beam cut)");
        return RNNTG_UNSUPPORTED;
      }
      if (flag == 4) {
        set_error("max_states binds above the device cap of 64 states per stream");
        return RNNTG_UNSUPPORTED;
      }
      if (flag == 6) {
        set_error("more than 32768 expansion candidates in one stream-frame (graph out-degree too high)");
        return RNNTG_UNSUPPORTED;
      }
      if (flag == 5) {
        set_error("best_path trace failed (inconsistent scores)");
        return RNNTG_INTERNAL;
      }
      if (flag != 0) {
        set_error("fsa kernel error flag " + std::to_string(flag));
        return RNNTG_INTERNAL;
      }
      break;
    }
  }
  st = finish(h, fs, B, out_mem, out_splits, out_tokens, out_scores, launches);
  if (st == RNNTG_OK) {
    h->last_fsa_fs.assign(fs, fs + B + 1);
    h->last_fsa_K = std::min(p->max_states, rnntg::kFsaMaxStates);
  }
  return st;
}

// ---- FSA step API (the reference's Algorithm-1 cycle, fsa_search.hpp:95-297) ----
namespace {
rnntg_status fsa_flag_status(int32_t flag) {
  switch (flag) {
    case 0:
      return RNNTG_OK;
    case 2:
      set_error("more than 32 distinct contexts per CTA frame (max_contexts too large for this build)");
      return RNNTG_UNSUPPORTED;
    case 3:
      set_error("candidate hash overflow (too many exact-score duplicates near the beam cut)");
      return RNNTG_UNSUPPORTED;
    case 4:
      set_error("max_states binds above the device cap of 64 states per stream");
      return RNNTG_UNSUPPORTED;
    case 6:
      set_error("more than 32768 expansion candidates in one stream-frame (graph out-degree too high)");
      return RNNTG_UNSUPPORTED;
    case 7:
      set_error("expand_arcs: stale get_contexts data");
      return RNNTG_INTERNAL;
    default:
      set_error("fsa kernel error flag " + std::to_string(flag));
      return RNNTG_INTERNAL;
  }
}

rnntg::FsaStepArgs step_args(rnntg_model_t h) {
  rnntg::FsaStepArgs a{};
  a.B = static_cast<int32_t>(h->step_fs.size()) - 1;
  a.V = h->d.V;
  a.frame_splits = h->splits.as<int32_t>();
  a.row_splits = h->step_rsplits.as<int32_t>();
  a.P = h->step_P.as<double>();
  a.graph_arcs = h->step_graph->arcs;
  a.graph_splits = h->step_graph->splits;
  a.graph_maxw = h->step_graph->maxw;
  a.beam = h->step_params.beam;
  a.max_states = h->step_params.max_states;
  a.max_contexts = h->step_params.max_contexts;
  a.lattice = h->lattice.ptr;
  a.lattice_cap = static_cast<int64_t>(h->lattice.bytes / 24);
  a.lattice_count = reinterpret_cast<unsigned long long*>(h->flag.as<char>() + 8);
  a.lat_frame_info = h->finfo.as<int32_t>();
  a.node_best = h->nodebest.as<double>();
  a.node_ctx = h->nodectx.as<int32_t>();
  a.state = h->step_state.ptr;
  a.tokens = h->tok.as<int32_t>();
  a.lengths = h->len.as<int32_t>();
  a.scores = h->score.as<double>();
  a.counters = h->counters.as<unsigned long long>();
  a.error_flag = h->flag.as<int32_t>();
  return a;
}
}  // namespace

rnntg_status rnntg_fsa_stream_begin(rnntg_model_t h, rnntg_graph_t graph, const rnntg_fsa_params* p, int32_t B,
                                    const int32_t* num_frames) {
  Nvtx nvtx_range("rnntg_fsa_stream_begin");
  if (!h || !p || !graph) return invalid("null argument");
  if (graph->model != h) return invalid("graph belongs to another model handle");
  // check_fsa_search_params (fsa_search.hpp:83-90), init_streams (95-120).
  if (!(p->beam >= 0.0)) return invalid("fsa search beam must be >= 0");
  if (p->max_states < 1) return invalid("max_states must be >= 1");
  if (p->max_contexts < 1) return invalid("max_contexts must be >= 1");
  if (B < 0 || (B > 0 && !num_frames)) return invalid("bad stream count");
  for (int32_t i = 0; i < B; ++i)
    if (num_frames[i] < 0) return invalid("num_frames must be >= 0");
  std::lock_guard<std::mutex> lk(h->mu);
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  h->last_fsa_fs.clear();
  h->step_open = false;
  h->step_have_rows = false;
  h->step_fs.assign(B + 1, 0);
  for (int32_t i = 0; i < B; ++i) h->step_fs[i + 1] = h->step_fs[i] + num_frames[i];
  const int64_t total = h->step_fs[B];
  const int K = std::min(p->max_states, rnntg::kFsaMaxStates);
  RNNTG_CUDA_TRY(h->splits.ensure(sizeof(int32_t) * (B + 1)));
  RNNTG_CUDA_TRY(cudaMemcpyAsync(h->splits.ptr, h->step_fs.data(), sizeof(int32_t) * (B + 1),
                                 cudaMemcpyHostToDevice, h->stream));
  RNNTG_CUDA_TRY(h->finfo.ensure(sizeof(int32_t) * 4 * (total + B)));
  RNNTG_CUDA_TRY(h->nodebest.ensure(sizeof(double) * (total * K + B)));
  RNNTG_CUDA_TRY(h->nodectx.ensure(sizeof(int32_t) * (total * K + B)));
  RNNTG_CUDA_TRY(h->lattice.ensure(sizeof(char) * 24 * std::max<int64_t>(int64_t{1} << 16, total * (2 * K + 8))));
  RNNTG_CUDA_TRY(h->flag.ensure(16));
  RNNTG_CUDA_TRY(cudaMemsetAsync(h->flag.ptr, 0, 16, h->stream));
  RNNTG_CUDA_TRY(h->counters.ensure(sizeof(unsigned long long) * 16));
  RNNTG_CUDA_TRY(cudaMemsetAsync(h->counters.ptr, 0, sizeof(unsigned long long) * 16, h->stream));
  RNNTG_CUDA_TRY(h->tok.ensure(sizeof(int32_t) * std::max<int64_t>(1, total)));
  RNNTG_CUDA_TRY(h->len.ensure(sizeof(int32_t) * std::max(1, B)));
  RNNTG_CUDA_TRY(h->score.ensure(sizeof(double) * std::max(1, B)));
  RNNTG_CUDA_TRY(h->step_state.ensure(sizeof(rnntg::FsaStepState) * std::max(1, B)));
  std::vector<rnntg::FsaStepState> st(std::max(1, B));
  for (int32_t i = 0; i < B; ++i) {
    rnntg::FsaStepState& x = st[i];
    std::memset(&x, 0, sizeof(x));
    x.n_act = 1;  // ((0,0), state 0, score 0, node 0)
    x.num_nodes = 1;
    x.T = num_frames[i];
  }
  RNNTG_CUDA_TRY(cudaMemcpyAsync(h->step_state.ptr, st.data(), sizeof(rnntg::FsaStepState) * std::max(1, B),
                                 cudaMemcpyHostToDevice, h->stream));
  RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->step_graph = graph;
  h->step_params = *p;
  h->step_open = true;
  return RNNTG_OK;
}

rnntg_status rnntg_fsa_stream_contexts(rnntg_model_t h, int32_t* out_row_splits, int32_t capacity,
                                       int32_t* out_contexts) {
  Nvtx nvtx_range("rnntg_fsa_stream_contexts");
  if (!h || !out_row_splits) return invalid("null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  if (!h->step_open) return invalid("no open FSA stream decode (rnntg_fsa_stream_begin)");
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  const int32_t B = static_cast<int32_t>(h->step_fs.size()) - 1;
  std::vector<rnntg::FsaStepState> st(std::max(1, B));
  if (B > 0)
    RNNTG_CUDA_TRY(cudaMemcpy(st.data(), h->step_state.ptr, sizeof(rnntg::FsaStepState) * B,
                              cudaMemcpyDeviceToHost));
  // get_contexts (fsa_search.hpp:124-154): done streams contribute none.
  std::vector<int32_t> ctx;
  h->step_rows.assign(B + 1, 0);
  h->step_nact.assign(B, 0);
  for (int32_t i = 0; i < B; ++i) {
    const rnntg::FsaStepState& x = st[i];
    int32_t n = 0;
    if (x.t < x.T) {
      h->step_nact[i] = x.n_act;
      for (int32_t j = 0; j < x.n_act; ++j)
        if (j == 0 || x.act_ctx[j] != x.act_ctx[j - 1]) {
          ctx.push_back(x.act_ctx[j]);
          ++n;
        }
    }
    h->step_rows[i + 1] = h->step_rows[i] + n;
  }
  std::memcpy(out_row_splits, h->step_rows.data(), sizeof(int32_t) * (B + 1));
  h->step_have_rows = true;
  if (capacity == 0) return RNNTG_OK;
  if (capacity < static_cast<int32_t>(ctx.size()) || !out_contexts) return invalid("contexts capacity too small");
  std::memcpy(out_contexts, ctx.data(), sizeof(int32_t) * ctx.size());
  return RNNTG_OK;
}

rnntg_status rnntg_fsa_stream_step(rnntg_model_t h, const double* logprobs, int32_t mem) {
  Nvtx nvtx_range("rnntg_fsa_stream_step");
  if (!h) return invalid("null model");
  if (mem != RNNTG_MEM_HOST && mem != RNNTG_MEM_DEVICE) return invalid("bad mem kind");
  std::lock_guard<std::mutex> lk(h->mu);
  if (!h->step_open) return invalid("no open FSA stream decode (rnntg_fsa_stream_begin)");
  if (!h->step_have_rows) {  // expand_arcs without a fresh get_contexts
    set_error("expand_arcs: stale get_contexts data");
    return RNNTG_INTERNAL;
  }
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  const int32_t B = static_cast<int32_t>(h->step_fs.size()) - 1;
  const int64_t rows = h->step_rows[B];
  if (rows > 0 && !logprobs) return invalid("logprobs is null");
  // Lattice room for this frame's worst case (every candidate kept as an
  // arc: n_act x (1 + out-degree) per stream); grown keeping the arcs so far.
  unsigned long long used = 0;
  RNNTG_CUDA_TRY(cudaMemcpy(&used, h->flag.as<char>() + 8, sizeof(used), cudaMemcpyDeviceToHost));
  int64_t worst = 0;
  for (int32_t i = 0; i < B; ++i) worst += static_cast<int64_t>(h->step_nact[i]) * (1 + h->step_graph->max_out);
  const size_t need = static_cast<size_t>(used + worst) * 24;
  if (need > h->lattice.bytes) RNNTG_CUDA_TRY(h->lattice.grow_keep(need * 2, used * 24, h->stream));
  const double* P = logprobs;
  if (mem == RNNTG_MEM_HOST && rows > 0) {
    RNNTG_CUDA_TRY(h->step_P.ensure(sizeof(double) * rows * h->d.V));
    RNNTG_CUDA_TRY(cudaMemcpyAsync(h->step_P.ptr, logprobs, sizeof(double) * rows * h->d.V, cudaMemcpyHostToDevice,
                                   h->stream));
    P = h->step_P.as<double>();
  }
  RNNTG_CUDA_TRY(cudaMemcpyAsync(h->splits.ptr, h->step_fs.data(), sizeof(int32_t) * (B + 1),
                                 cudaMemcpyHostToDevice, h->stream));  // the handle may have decoded meanwhile
  RNNTG_CUDA_TRY(h->step_rsplits.ensure(sizeof(int32_t) * (B + 1)));
  RNNTG_CUDA_TRY(cudaMemcpyAsync(h->step_rsplits.ptr, h->step_rows.data(), sizeof(int32_t) * (B + 1),
                                 cudaMemcpyHostToDevice, h->stream));
  rnntg::FsaStepArgs a = step_args(h);
  a.P = P;
  RNNTG_CUDA_TRY(rnntg::launch_fsa_step(a, false, h->stream));
  int32_t flag = 0;
  RNNTG_CUDA_TRY(cudaMemcpyAsync(&flag, h->flag.ptr, sizeof(flag), cudaMemcpyDeviceToHost, h->stream));
  RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->step_have_rows = false;
  if (flag) {
    h->step_open = false;  // the decode state is no longer consistent
    return fsa_flag_status(flag);
  }
  return RNNTG_OK;
}

rnntg_status rnntg_fsa_stream_end(rnntg_model_t h, int32_t* out_splits, int32_t* out_tokens, double* out_scores) {
  Nvtx nvtx_range("rnntg_fsa_stream_end");
  if (!h || !out_splits) return invalid("null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  if (!h->step_open) return invalid("no open FSA stream decode (rnntg_fsa_stream_begin)");
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  const std::vector<int32_t> fs = h->step_fs;
  const int32_t B = static_cast<int32_t>(fs.size()) - 1;
  RNNTG_CUDA_TRY(h->splits.ensure(sizeof(int32_t) * (B + 1)));
  RNNTG_CUDA_TRY(cudaMemcpyAsync(h->splits.ptr, fs.data(), sizeof(int32_t) * (B + 1), cudaMemcpyHostToDevice,
                                 h->stream));
  RNNTG_CUDA_TRY(cudaEventRecord(h->ev[0], h->stream));
  RNNTG_CUDA_TRY(cudaEventRecord(h->ev[1], h->stream));
  RNNTG_CUDA_TRY(rnntg::launch_fsa_step(step_args(h), true, h->stream));
  int32_t flag = 0;
  RNNTG_CUDA_TRY(cudaMemcpyAsync(&flag, h->flag.ptr, sizeof(flag), cudaMemcpyDeviceToHost, h->stream));
  RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (flag == 5) {
    set_error("best_path trace failed (inconsistent scores)");
    return RNNTG_INTERNAL;
  }
  h->pipelined = false;
  rnntg_status st = finish(h, fs.data(), B, RNNTG_MEM_HOST, out_splits, out_tokens, out_scores, 1);
  if (st) return st;
  h->step_open = false;
  h->last_fsa_fs = fs;
  h->last_fsa_K = std::min(h->step_params.max_states, rnntg::kFsaMaxStates);
  return RNNTG_OK;
}

rnntg_status rnntg_fsa_lattice(rnntg_model_t h, int32_t s, int32_t* num_nodes, int32_t* num_arcs,
                               int32_t capacity, int32_t* src, int32_t* dst, int32_t* label,
                               double* score) {
  if (!h || !num_nodes || !num_arcs) return invalid("null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->last_fsa_fs.empty()) return invalid("no fsa_beam_search has run on this handle");
  const int32_t B = static_cast<int32_t>(h->last_fsa_fs.size()) - 1;
  if (s < 0 || s >= B) return invalid("stream index out of range");
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  const int32_t f0 = h->last_fsa_fs[s], T = h->last_fsa_fs[s + 1] - f0;
  struct I4 {
    int32_t off, cnt, base, n;
  };
  struct Arc24 {
    int32_t src, dst, label, pad;
    double score;
  };
  std::vector<I4> fi(std::max(1, T));
  if (T > 0)
    RNNTG_CUDA_TRY(cudaMemcpy(fi.data(), h->finfo.as<int32_t>() + 4 * (static_cast<int64_t>(f0) + s),
                              sizeof(I4) * T, cudaMemcpyDeviceToHost));
  // build_lattice (fsa_search.hpp:309-317): frame layers, then the hops from
  // the final-frame nodes into the super-final node.
  const int32_t nn = T == 0 ? 1 : fi[T - 1].base + fi[T - 1].n;
  const int32_t first_final = T == 0 ? 0 : fi[T - 1].base;
  const int32_t n_final = T == 0 ? 1 : fi[T - 1].n;
  int64_t total = n_final;
  for (int32_t t = 0; t < T; ++t) total += fi[t].cnt;
  *num_nodes = nn + 1;
  *num_arcs = static_cast<int32_t>(total);
  if (capacity == 0) return RNNTG_OK;
  if (capacity < total || !src || !dst || !label || !score) return invalid("lattice capacity too small");
  std::vector<Arc24> buf;
  int64_t k = 0;
  for (int32_t t = 0; t < T; ++t) {
    if (fi[t].cnt == 0) continue;
    buf.resize(fi[t].cnt);
    RNNTG_CUDA_TRY(cudaMemcpy(buf.data(), h->lattice.as<char>() + static_cast<int64_t>(fi[t].off) * 24,
                              sizeof(Arc24) * fi[t].cnt, cudaMemcpyDeviceToHost));
    for (const Arc24& a : buf) {
      src[k] = a.src;
      dst[k] = a.dst;
      label[k] = a.label;
      score[k] = a.score;
      ++k;
    }
  }
  for (int32_t i = 0; i < n_final; ++i, ++k) {
    src[k] = first_final + i;
    dst[k] = nn;
    label[k] = 0;
    score[k] = 0.0;
  }
  return RNNTG_OK;
}

rnntg_status rnntg_fsa_lattice_best(rnntg_model_t h, int32_t merge_op, int32_t nbest_n, uint64_t seed,
                                    int32_t* out_splits, int32_t* out_tokens, double* out_logprob) {
  Nvtx nvtx_range("rnntg_fsa_lattice_best");
  if (!h || !out_splits) return invalid("null argument");
  if (merge_op != RNNTG_MERGE_LOG_ADD)
    return invalid("rnntg_fsa_lattice_best: kMax best sequences are rnntg_fsa_beam_search's own output");
  if (nbest_n < 1) return invalid("nbest_n must be >= 1");  // fsa_search.hpp:411
  if (nbest_n > 1024) {
    set_error("nbest_n > 1024 is beyond this build's per-stream path cap");
    return RNNTG_UNSUPPORTED;
  }
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->last_fsa_fs.empty()) return invalid("no fsa_beam_search has run on this handle");
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  const std::vector<int32_t>& fs = h->last_fsa_fs;
  const int32_t B = static_cast<int32_t>(fs.size()) - 1;
  const int64_t total = fs[B];
  int32_t tmax = 0;
  for (int32_t i = 0; i < B; ++i) tmax = std::max(tmax, fs[i + 1] - fs[i]);
  const int32_t K = h->last_fsa_K;
  out_splits[0] = 0;
  if (B == 0) return RNNTG_OK;
  // DetRng(seed).uniform01() stream: nbest paths x (T + 2) draws (every
  // complete path of these layered lattices visits T + 2 states).
  const int64_t nu = static_cast<int64_t>(nbest_n) * (tmax + 2);
  if (h->ladd_seed != seed || h->ladd_n < nu) {
    RNNTG_CUDA_TRY(h->ladd_u.ensure(sizeof(double) * nu));
    RNNTG_CUDA_TRY(rnntg::launch_mt19937_64_uniforms(seed, nu, h->ladd_u.as<double>(), h->stream));
    h->ladd_seed = seed;
    h->ladd_n = nu;
  }
  RNNTG_CUDA_TRY(h->splits.ensure(sizeof(int32_t) * (B + 1)));
  RNNTG_CUDA_TRY(cudaMemcpyAsync(h->splits.ptr, fs.data(), sizeof(int32_t) * (B + 1), cudaMemcpyHostToDevice,
                                 h->stream));
  RNNTG_CUDA_TRY(h->ladd_tot.ensure(sizeof(double) * (total * K + B)));
  RNNTG_CUDA_TRY(h->ladd_narc.ensure(sizeof(int2) * (total * K + B)));
  RNNTG_CUDA_TRY(h->ladd_paths.ensure(sizeof(int32_t) * nbest_n * (total + B)));
  RNNTG_CUDA_TRY(h->ladd_pos.ensure(sizeof(int32_t) * B * rnntg::kLogAddWarps * 3 * (tmax + 2)));
  RNNTG_CUDA_TRY(h->tok.ensure(sizeof(int32_t) * std::max<int64_t>(1, total)));
  RNNTG_CUDA_TRY(h->len.ensure(sizeof(int32_t) * B));
  RNNTG_CUDA_TRY(h->score.ensure(sizeof(double) * B));
  RNNTG_CUDA_TRY(h->flag.ensure(16));
  for (int attempt = 0;; ++attempt) {
    RNNTG_CUDA_TRY(h->ladd_cells.ensure(sizeof(double) * B * rnntg::kLogAddWarps * 2 * h->ladd_cell_cap));
    RNNTG_CUDA_TRY(cudaMemsetAsync(h->flag.ptr, 0, 16, h->stream));
    rnntg::LogAddArgs a{};
    a.B = B;
    a.V = h->d.V;
    a.K = K;
    a.nbest = nbest_n;
    a.frame_splits = h->splits.as<int32_t>();
    a.lattice = h->lattice.ptr;
    a.lat_frame_info = h->finfo.as<int32_t>();
    a.node_ctx = h->nodectx.as<int32_t>();
    a.uniforms = h->ladd_u.as<double>();
    a.tot = h->ladd_tot.as<double>();
    a.node_arcs = h->ladd_narc.as<int2>();
    a.paths = h->ladd_paths.as<int32_t>();
    a.cells = h->ladd_cells.as<double>();
    a.pos = h->ladd_pos.as<int32_t>();
    a.cell_cap = h->ladd_cell_cap;
    a.tmax = tmax;
    a.tokens = h->tok.as<int32_t>();
    a.lengths = h->len.as<int32_t>();
    a.logprob = h->score.as<double>();
    a.error_flag = h->flag.as<int32_t>();
    RNNTG_CUDA_TRY(rnntg::launch_lattice_logadd(a, h->stream));
    int32_t flag = 0;
    RNNTG_CUDA_TRY(cudaMemcpyAsync(&flag, h->flag.ptr, sizeof(flag), cudaMemcpyDeviceToHost, h->stream));
    RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (flag == 0) break;
    if (attempt >= 6) {
      set_error("log-add product DP scratch could not be sized");
      return RNNTG_INTERNAL;
    }
    h->ladd_cell_cap *= 4;  // a layer of the intersection held more cells: regrow and rerun
  }
  std::vector<int32_t> lens(B);
  RNNTG_CUDA_TRY(cudaMemcpy(lens.data(), h->len.ptr, sizeof(int32_t) * B, cudaMemcpyDeviceToHost));
  for (int32_t i = 0; i < B; ++i) out_splits[i + 1] = out_splits[i] + lens[i];
  const int64_t ntok = out_splits[B];
  if (ntok > 0) {
    if (!out_tokens) return invalid("out_tokens is null");
    RNNTG_CUDA_TRY(h->out_splits.ensure(sizeof(int32_t) * (B + 1)));
    RNNTG_CUDA_TRY(h->out_tok.ensure(sizeof(int32_t) * ntok));
    RNNTG_CUDA_TRY(cudaMemcpyAsync(h->out_splits.ptr, out_splits, sizeof(int32_t) * (B + 1),
                                   cudaMemcpyHostToDevice, h->stream));
    compact_tokens_kernel<<<B, 128, 0, h->stream>>>(h->tok.as<int32_t>(), h->splits.as<int32_t>(),
                                                    h->out_splits.as<int32_t>(), B, 1, h->out_tok.as<int32_t>());
    RNNTG_CUDA_TRY(cudaGetLastError());
    RNNTG_CUDA_TRY(cudaMemcpyAsync(out_tokens, h->out_tok.ptr, sizeof(int32_t) * ntok, cudaMemcpyDeviceToHost,
                                   h->stream));
  }
  if (out_logprob)
    RNNTG_CUDA_TRY(cudaMemcpyAsync(out_logprob, h->score.ptr, sizeof(double) * B, cudaMemcpyDeviceToHost,
                                   h->stream));
  RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return RNNTG_OK;
}

rnntg_status rnntg_fsa_lattice_text(rnntg_model_t h, int32_t s, int32_t with_header, char* buf,
                                    int64_t capacity, int64_t* length) {
  if (!h || !length) return invalid("null argument");
  int32_t nn = 0, na = 0;
  rnntg_status st = rnntg_fsa_lattice(h, s, &nn, &na, 0, nullptr, nullptr, nullptr, nullptr);
  if (st) return st;
  std::vector<int32_t> src(std::max(1, na)), dst(std::max(1, na)), lab(std::max(1, na));
  std::vector<double> sc(std::max(1, na));
  if ((st = rnntg_fsa_lattice(h, s, &nn, &na, na, src.data(), dst.data(), lab.data(), sc.data()))) return st;
  // serialize_lattice (fsa_search.hpp:429-435) over serialize_fsa_text
  // (fsa.hpp:243-262): "src dst label score" per arc, then "state score" per
  // final, scores in the shortest round-trip form of std::to_chars
  // (detail::format_score, fsa.hpp:127-131).
  std::string out;
  out.reserve(static_cast<size_t>(na) * 32 + 64);
  auto score = [&out](double v) {
    char b[64];
    const auto r = std::to_chars(b, b + sizeof(b), v);
    out.append(b, r.ptr);
  };
  if (with_header) {
    int32_t T = 0;
    {
      std::lock_guard<std::mutex> lk(h->mu);
      T = h->last_fsa_fs[s + 1] - h->last_fsa_fs[s];
    }
    out += "# stream=" + std::to_string(s) + " frames=" + std::to_string(T) + "\n";
  }
  for (int32_t i = 0; i < na; ++i) {
    out += std::to_string(src[i]);
    out += ' ';
    out += std::to_string(dst[i]);
    out += ' ';
    out += std::to_string(lab[i]);
    out += ' ';
    score(sc[i]);
    out += '\n';
  }
  out += std::to_string(nn - 1);  // the super-final node, final score 0
  out += ' ';
  score(0.0);
  out += '\n';
  *length = static_cast<int64_t>(out.size());
  if (capacity == 0) return RNNTG_OK;
  if (!buf || capacity < *length + 1) return invalid("lattice text capacity too small");
  std::memcpy(buf, out.data(), out.size());
  buf[out.size()] = '\0';
  return RNNTG_OK;
}

rnntg_status rnntg_model_set_encoder(rnntg_model_t h, const rnntg_encoder_desc* e) {
  if (!h || !e) return invalid("null argument");
  if (e->feat_dim < 1) return invalid("model dims must be >= 1");
  if (!e->enc_w1 || !e->enc_b1 || !e->enc_w2 || !e->enc_b2) return invalid("encoder weight pointer is null");
  std::lock_guard<std::mutex> lk(h->mu);
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  rnntg::DeviceModel& d = h->d;
  const int32_t D = d.D, F = e->feat_dim, Dp = round_up(D, 128);
  rnntg_status st;
  if ((st = upload(h, &d.enc_w1t, transpose_pad(e->enc_w1, D, F, Dp))) ||
      (st = upload(h, &d.enc_b1, std::vector<float>(e->enc_b1, e->enc_b1 + D))) ||
      (st = upload(h, &d.enc_w2t, transpose_pad(e->enc_w2, D, D, Dp))) ||
      (st = upload(h, &d.enc_b2, std::vector<float>(e->enc_b2, e->enc_b2 + D))))
    return st;
  d.F = F;
  return RNNTG_OK;
}

rnntg_status rnntg_encoder_forward(rnntg_model_t h, const float* feats, const int32_t* fs,
                                   int32_t B, int32_t mem, float* enc_out) {
  Nvtx nvtx_range("rnntg_encoder_forward");
  if (!h) return invalid("null model");
  if (h->d.F == 0) return invalid("no encoder weights (rnntg_model_set_encoder)");
  if (mem != RNNTG_MEM_HOST && mem != RNNTG_MEM_DEVICE) return invalid("bad mem kind");
  rnntg_status st = check_frames(feats, fs, B);
  if (st) return st;
  const int64_t total = B > 0 ? fs[B] : 0;
  if (total == 0) return RNNTG_OK;
  if (!enc_out) return invalid("enc_out is null");
  std::lock_guard<std::mutex> lk(h->mu);
  return encoder_impl(h, feats, fs, B, mem, enc_out);
}


rnntg_status rnntg_debug_decoder_projection(rnntg_model_t h, const int32_t* ctxs,
                                            int32_t n, float* pd_out) {
  if (!h || (n > 0 && (!ctxs || !pd_out))) return invalid("null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  const int32_t J = h->d.J;
  for (int32_t i = 0; i < n; ++i) {
    if (ctxs[i] < 0 || ctxs[i] >= h->d.V * h->d.V) return invalid("packed context out of range");
    RNNTG_CUDA_TRY(cudaMemcpyAsync(pd_out + static_cast<size_t>(i) * J,
                                   h->d.pd_table + static_cast<size_t>(ctxs[i]) * J,
                                   sizeof(float) * J, cudaMemcpyDeviceToHost, h->stream));
  }
  RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return RNNTG_OK;
}

rnntg_status rnntg_debug_joiner_logits(rnntg_model_t h, const float* enc,
                                       const int32_t* ctxs, int32_t n,
                                       float* logits_out) {
  if (!h || (n > 0 && (!enc || !ctxs || !logits_out))) return invalid("null argument");
  if (n <= 0) return RNNTG_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  RNNTG_CUDA_TRY(cudaSetDevice(h->device));
  for (int32_t i = 0; i < n; ++i)
    if (ctxs[i] < 0 || ctxs[i] >= h->d.V * h->d.V) return invalid("packed context out of range");
  const int32_t D = h->d.D, J = h->d.J, V = h->d.V;
  RNNTG_CUDA_TRY(h->enc.ensure(sizeof(float) * n * D));
  RNNTG_CUDA_TRY(h->pe.ensure(sizeof(float) * n * J));
  RNNTG_CUDA_TRY(h->ctx.ensure(sizeof(int32_t) * n));
  RNNTG_CUDA_TRY(h->logits.ensure(sizeof(float) * n * V));
  RNNTG_CUDA_TRY(cudaMemcpyAsync(h->enc.ptr, enc, sizeof(float) * n * D, cudaMemcpyHostToDevice, h->stream));
  RNNTG_CUDA_TRY(cudaMemcpyAsync(h->ctx.ptr, ctxs, sizeof(int32_t) * n, cudaMemcpyHostToDevice, h->stream));
  RNNTG_CUDA_TRY(rnntg::launch_gemm_exact(h->enc.as<float>(), D, h->d.j_wet, h->d.Jp, nullptr,
                                          h->pe.as<float>(), J, n, J, D, false, nullptr, 0, 0,
                                          h->stream));
  RNNTG_CUDA_TRY(rnntg::launch_joiner_rows_exact(h->d, h->pe.as<float>(), h->ctx.as<int32_t>(), n,
                                                 h->logits.as<float>(), h->stream));
  RNNTG_CUDA_TRY(cudaMemcpyAsync(logits_out, h->logits.ptr, sizeof(float) * n * V,
                                 cudaMemcpyDeviceToHost, h->stream));
  RNNTG_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return RNNTG_OK;
}

rnntg_status rnntg_debug_tanhf_chunk_hashes(int32_t device, int32_t first_chunk,
                                            int32_t num_chunks, uint64_t* hashes) {
  if (first_chunk < 0 || num_chunks < 1 || first_chunk + num_chunks > 256 || !hashes)
    return invalid("chunk range must lie in [0, 256)");
  RNNTG_CUDA_TRY(cudaSetDevice(device));
  unsigned long long* d = nullptr;
  RNNTG_CUDA_TRY(cudaMalloc(&d, sizeof(unsigned long long) * num_chunks));
  cudaError_t e = rnntg::launch_tanhf_hash(first_chunk, num_chunks, d, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess)
    e = cudaMemcpy(hashes, d, sizeof(unsigned long long) * num_chunks, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return RNNTG_CUDA_ERROR;
  }
  return RNNTG_OK;
}


rnntg_status rnntg_debug_log_softmax_lse(int32_t device, const float* logits, int32_t n, int32_t V,
                                         double* lse) {
  if (n < 0 || V < 1 || V > rnntg::kMaxVocab || (n > 0 && (!logits || !lse)))
    return invalid("bad log-softmax arguments");
  if (n == 0) return RNNTG_OK;
  return debug_roundtrip(device, logits, static_cast<size_t>(n) * V, lse, static_cast<size_t>(n),
                         [&](const float* di, double* dout) {
                           return rnntg::launch_log_softmax_rows(di, n, V, dout, nullptr);
                         });
}

rnntg_status rnntg_debug_f64_math(int32_t device, int32_t op, const double* x, int64_t n, double* y) {
  if (op < 0 || op > 3 || n < 0 || (n > 0 && (!x || !y))) return invalid("bad f64 math arguments");
  if (n == 0) return RNNTG_OK;
  return debug_roundtrip(device, x, static_cast<size_t>(n), y, static_cast<size_t>(n),
                         [&](const double* di, double* dout) { return rnntg::launch_f64_math(op, di, n, dout, nullptr); });
}

}  // extern "C"
