// Internal declarations shared by the rnntg CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/rnntg.h"

namespace rnntg {

constexpr int kMaxVocab = 512;      // joiner output row staged whole in smem
constexpr int kMaxJoiner = 512;     // reference limit (model.hpp:287-288)
constexpr int kMaxBeam = 8;         // hypotheses per stream (warp lanes)
constexpr int kFsaMaxStates = 64;   // FSA active tuples per stream
constexpr int kDecodeThreads = 512; // persistent decode CTA (16 warps)

void set_error(const std::string& msg);

#define RNNTG_CUDA_TRY(expr)                                              \
  do {                                                                    \
    cudaError_t _e = (expr);                                              \
    if (_e != cudaSuccess) {                                              \
      ::rnntg::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
      return RNNTG_CUDA_ERROR;                                            \
    }                                                                     \
  } while (0)

// Device copy of the model, laid out for the kernels.
struct DeviceModel {
  int32_t V = 0, D = 0, E = 0, J = 0;
  int32_t Vp = 0;          // V rounded up to a multiple of 128
  float* emb = nullptr;    // [V][E]
  float* ctx_wt = nullptr; // [2E][Ep]  (transposed ctx_w, k-major)
  float* ctx_b = nullptr;  // [E]
  float* j_wet = nullptr;  // [D][Jp]   (transposed j_we)
  float* j_wdt = nullptr;  // [E][Jp]   (transposed j_wd)
  float* j_b = nullptr;    // [J]
  float* out_wt = nullptr; // [J][Vp]   (transposed out_w, zero-padded)
  float* out_b = nullptr;  // [Vp]
  float* zeros = nullptr;  // [max(Vp, Jp)] zero bias (encoder projection starts from 0.0f)
  float* pd_table = nullptr; // [V*V][J]: decoder-side joiner projection of
                             // every packed context (K0)
  uint16_t* out_w_bf16 = nullptr; // bf16 out_w, UMMA chunk layout (tcgen05 variant)
  // optional encoder (rnntg_model_set_encoder): k-major transposed weights
  int32_t F = 0;
  float* enc_w1t = nullptr; // [F][Dp]
  float* enc_b1 = nullptr;  // [D]
  float* enc_w2t = nullptr; // [D][Dp]
  float* enc_b2 = nullptr;  // [D]
  int32_t Ep = 0, Jp = 0;
};

// Growable device scratch.
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&ptr, need);
    if (e == cudaSuccess) bytes = need;
    return e;
  }
  // grow to `need` bytes keeping the first `keep` bytes (stream-ordered copy)
  cudaError_t grow_keep(size_t need, size_t keep, cudaStream_t s) {
    if (need <= bytes) return cudaSuccess;
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, need);
    if (e != cudaSuccess) return e;
    if (ptr && keep) e = cudaMemcpyAsync(p, ptr, keep, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (ptr) cudaFree(ptr);
    ptr = p;
    bytes = need;
    return e;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
};

// ---- exact sequential GEMM (gemm_exact.cu) ----
// Y[m][n] = (bias ? bias[n] : 0) + sum_{k<K} X[m][k] * Wt[k][n], the k sum in
// index order with separately rounded products (the reference's affine,
// model.hpp:100-108).  Wt is [K][ldw] with ldw >= round_up(N, 128), padding
// columns zero.  If ctx_emb != nullptr, row m is the decoder input of packed
// context (ctx_base + m): [emb[c / V] ; emb[c % V]], K = 2E.
cudaError_t launch_gemm_exact(const float* X, int64_t ldx, const float* Wt,
                              int32_t ldw, const float* bias, float* Y,
                              int64_t ldy, int64_t M, int32_t N, int32_t K,
                              bool apply_tanh, const float* ctx_emb,
                              int32_t ctx_V, int64_t ctx_base,
                              cudaStream_t stream);
// The same over row groups: logical row m is physical row
// (m / grp) * gstride + m % grp of X and Y (M a multiple of grp): a time
// slice of grp frames of streams of uniform length gstride, X and Y offset
// to the slice's first frame.  grp = 0: contiguous rows.
cudaError_t launch_gemm_exact_grouped(const float* X, int64_t ldx, const float* Wt, int32_t ldw,
                                      const float* bias, float* Y, int64_t ldy, int64_t M, int32_t N,
                                      int32_t K, bool apply_tanh, const float* ctx_emb,
                                      int32_t ctx_V, int64_t ctx_base, int32_t grp, int64_t gstride,
                                      cudaStream_t stream);

// ---- persistent decode kernels (decode.cu) ----
struct DecodeArgs {
  const DeviceModel* m;     // host struct, copied by value into kernel params
  const float* pe;          // [sum T][J] encoder-side projections
  const int32_t* frame_splits; // device [B+1]
  int32_t B;
  int32_t streams_per_cta;
  int32_t* tokens;          // device [sum T] (per-stream slot at frame_splits)
  int32_t* lengths;         // device [B]
  double* scores;           // device [B]
  unsigned long long* counters; // device [8]
  // greedy: symbols per frame (1 = greedy_search_batch; > 1 = greedy_search)
  int32_t symbol_cap;
  int32_t count_capped;     // count frames stopped by the cap (S unlimited)
  // beam
  int32_t beam_size, merge_op, length_norm, max_total;
  int32_t joiner_bf16;      // 1: tcgen05 bf16 joiner variant (not token-exact)
  uint32_t* backptr;        // device [(sum T + B) * kMaxBeam]
  void* node_pool;          // beam S > 1: device int2 [(sum T * cap + B) * kMaxBeam] (parent, token) nodes
  // beam, time-sliced launches (host frames: the copy and K1 of slice k+1
  // overlap the decode of slice k): this launch decodes frames [t0, t1) of
  // every stream; hypothesis sets persist between launches in hyps_state.
  int32_t t0 = 0, t1 = 0x7fffffff;
  void* hyps_state = nullptr;  // device [B] beam hypothesis sets (beam_state_bytes() each)
  // fsa
  const void* graph_arcs;   // device int4-packed arcs
  const int32_t* graph_splits;
  const double* graph_maxw;     // device [states]: max outgoing arc weight (-inf if none)
  int32_t graph_states;
  double fsa_beam;
  int32_t max_states, max_contexts;
  void* lattice;            // device lattice arc pool
  int64_t lattice_cap;
  unsigned long long* lattice_count; // device arc pool bump counter
  int32_t* lat_frame_info;  // device int4 per (stream, frame): off, count, node base, nodes
  double* node_best;        // device per-node suffix scores (best_path)
  int32_t* node_ctx;        // device per-node packed context (lattice_to_best_seq(kLogAdd), logadd.cu)
  int32_t* error_flag;      // device
};

cudaError_t launch_decode_greedy(const DecodeArgs& a, cudaStream_t s);
size_t beam_state_bytes();  // per-stream hypothesis set carried between time-sliced launches
// small batches (<= 144 streams): thread-block clusters with out_w slices
// resident in shared memory (cluster.cu)
bool greedy_cluster_fits(const DeviceModel& d, int32_t B);
cudaError_t launch_decode_greedy_cluster(const DecodeArgs& a, cudaStream_t s);
cudaError_t launch_decode_beam(const DecodeArgs& a, cudaStream_t s);
// small batches (<= num_sms / 8 * 64 / beam streams): thread-block clusters
// with out_w column slices resident in shared memory (decode.cu); returns
// the streams per cluster, or 0 when the batch does not fit
int beam_cluster_streams(const DeviceModel& d, int32_t B, int32_t beam_size, int num_sms);
cudaError_t launch_decode_beam_cluster(const DecodeArgs& a, cudaStream_t s);
cudaError_t launch_decode_fsa(const DecodeArgs& a, cudaStream_t s);

// The FSA step API (fsa_search.hpp:95-297): per-stream state between steps
// (the reference's DecodeStream without its host vectors) and one launch
// per expand_arcs + prune_streams, or for the final best paths.
struct FsaStepState {
  int32_t n_act, num_nodes, t, T, flag, pad;
  int32_t act_ctx[kFsaMaxStates], act_state[kFsaMaxStates], act_node[kFsaMaxStates];
  double act_score[kFsaMaxStates];
};
struct FsaStepArgs {
  int32_t B, G, V;
  const int32_t* frame_splits;  // device [B+1]: each stream's num_frames, as splits
  const int32_t* row_splits;    // device [B+1]: the caller's log-prob rows of this step per stream
  const double* P;              // device [rows][V] log-prob rows (expand_arcs' logprobs)
  const void* graph_arcs;
  const int32_t* graph_splits;
  const double* graph_maxw;
  double beam;
  int32_t max_states, max_contexts;
  void* lattice;
  int64_t lattice_cap;
  unsigned long long* lattice_count;
  int32_t* lat_frame_info;
  double* node_best;
  int32_t* node_ctx;
  void* state;                  // device FsaStepState [B]
  int32_t* tokens;              // device [sum T] (finish)
  int32_t* lengths;             // device [B] (finish)
  double* scores;               // device [B] (finish)
  unsigned long long* counters; // device [16]
  int32_t* error_flag;
};
cudaError_t launch_fsa_step(FsaStepArgs a, bool finish, cudaStream_t s);

// lattice_to_best_seq(kLogAdd) (fsa_search.hpp:410-425) on the device
// lattices of the last FSA decode (logadd.cu).
struct LogAddArgs {
  int32_t B, V, K, nbest;
  const int32_t* frame_splits;   // device [B+1]
  const void* lattice;           // device LatArc pool
  const int32_t* lat_frame_info; // device int4 per (stream, frame)
  const int32_t* node_ctx;       // device, indexed like node_best
  const double* uniforms;        // device [nbest * (Tmax + 2)]: DetRng(seed).uniform01() in order
  double* tot;                   // scratch, indexed like node_best: log-semiring suffix totals
  int2* node_arcs;               // scratch, indexed like node_best: {first arc, count} (-1: the super-final hop)
  int32_t* paths;                // scratch [nbest * (sum T + B)] sampled blank-free label sequences
  double* cells;                 // scratch [B * kLogAddWarps * 2 * cell_cap] DP layers
  int32_t* pos;                  // scratch [B * kLogAddWarps * 3 * (Tmax + 2)] sorted positions
  int64_t cell_cap;
  int32_t tmax;
  int32_t* tokens;               // device [sum T]: best sequence at frame_splits[i]
  int32_t* lengths;              // device [B]
  double* logprob;               // device [B]: its total log-probability (-inf: no path)
  int32_t* error_flag;           // device: 1 = cell scratch too small
};
constexpr int kLogAddWarps = 8;
cudaError_t launch_mt19937_64_uniforms(uint64_t seed, int64_t n, double* out, cudaStream_t s);
cudaError_t launch_lattice_logadd(const LogAddArgs& a, cudaStream_t s);
int decode_num_sms(int device);
int decode_num_sms_current();

cudaError_t launch_log_softmax_rows(const float* logits, int32_t n, int32_t V, double* lse, cudaStream_t s);
cudaError_t launch_f64_math(int32_t op, const double* x, int64_t n, double* y, cudaStream_t s);
cudaError_t launch_tanhf_hash(int32_t first_chunk, int32_t num_chunks,
                              unsigned long long* d_hashes, cudaStream_t s);
cudaError_t launch_joiner_rows_exact(const DeviceModel& m, const float* pe,
                                     const int32_t* ctxs, int32_t n,
                                     float* logits, cudaStream_t s);

}  // namespace rnntg
