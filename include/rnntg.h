/*
 * rnntg — B200 (sm_100a) one-symbol-per-frame transducer decoding.
 *
 * Plain C ABI over the CUDA library paper_2211_00484_b200/librnntg.so.
 * No torch types, no C++ types: pointers, sizes and POD parameter structs.
 *
 * Each entry point replaces one public function of the reference C++ library
 * (rnnt-kit, /root/reference/proj/include/rnnt):
 *
 *   rnntg_model_create          <- init_model / ToyTransducer weights
 *                                  (model.hpp:61-90, 129-169; weights in
 *                                  param_views naming, model.hpp:75-82)
 *   rnntg_greedy_search_batch   <- greedy_search_batch   (search.hpp:107-167)
 *   rnntg_greedy_search         <- greedy_search, any S  (search.hpp:76-100),
 *                                  batched over utterances
 *   rnntg_beam_search_batch     <- beam_search, S = 1    (search.hpp:206-277),
 *                                  batched over utterances like the CLI's
 *                                  parallel_for (tools/rnnt_main.cpp:274-287)
 *   rnntg_graph_create          <- Fsa / make_fsa        (fsa.hpp:54-111)
 *   rnntg_fsa_beam_search       <- fsa_beam_search       (fsa_search.hpp:326-387)
 *                                  + lattice_to_best_seq(kMax) (394-409)
 *                                  + best_path(...).score (fsa.hpp:345-376)
 *
 * The reference takes acoustic features and runs its toy encoder inside the
 * search; the north-star boundary takes encoder frames (the encoder is the
 * caller's).  include/rnnt_gpu.hpp restores the exact
 * reference signatures on top of this ABI by running the reference encoder
 * on the host first.
 *
 * Errors: every call returns an rnntg_status; rnntg_last_error() gives the
 * message of the calling thread's last failure.  INVALID_ARGUMENT is the
 * reference's ValidationError; INTERNAL is its std::logic_error.
 *
 * Threading: a model handle owns one CUDA device, one CUDA stream and its
 * scratch memory; calls on a handle are serialised, different handles may be
 * used from different threads.  Graph handles are read-only once created and
 * may be shared by the decode calls of the handle they were created on.
 */
#ifndef RNNTG_H_
#define RNNTG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RNNTG_OK = 0,
  RNNTG_INVALID_ARGUMENT = 1, /* reference ValidationError */
  RNNTG_INTERNAL = 2,         /* reference std::logic_error */
  RNNTG_CUDA_ERROR = 3,
  RNNTG_UNSUPPORTED = 4       /* valid for the reference, beyond a device cap */
} rnntg_status;

/* Where the frame / result buffers of a decode call live. */
typedef enum {
  RNNTG_MEM_HOST = 0,   /* host memory: H2D and D2H copies inside the call */
  RNNTG_MEM_DEVICE = 1, /* device memory on the model's GPU */
  /* search inputs only: `enc` points to host ACOUSTIC FEATURES [sum T][F]
   * (the reference API's input); the GPU encoder (rnntg_encoder_forward,
   * bit-exact encoder_forward) turns them into device-resident frames first.
   * Needs rnntg_model_set_encoder.  Outputs are host memory. */
  RNNTG_MEM_HOST_FEATURES = 2
} rnntg_mem;

typedef enum { RNNTG_MERGE_MAX = 0, RNNTG_MERGE_LOG_ADD = 1 } rnntg_merge_op;

/* Joiner arithmetic.  EXACT reproduces the reference's fp32 logits bit for
 * bit (sequential non-fused fp32 on CUDA cores + a glibc-2.39 tanhf port).
 * BF16 runs the output projection on tcgen05 tensor cores with bf16 operands
 * and fp32 accumulation; it is the separately reported fast variant and is
 * NOT token-exact. */
typedef enum { RNNTG_JOINER_EXACT = 0, RNNTG_JOINER_BF16 = 1 } rnntg_joiner_mode;

typedef struct rnntg_model_s* rnntg_model_t;
typedef struct rnntg_graph_s* rnntg_graph_t;

/* Stateless-transducer weights, fp32 row-major host arrays in the
 * reference's param_views naming (model.hpp:75-82).  context_size must be 2. */
typedef struct {
  int32_t vocab_size;   /* V, blank = 0 */
  int32_t enc_dim;      /* D */
  int32_t emb_dim;      /* E */
  int32_t joiner_dim;   /* J (<= 512, as model.hpp:287-288) */
  int32_t context_size; /* must be 2 */
  const float* emb;     /* [V][E]   */
  const float* ctx_w;   /* [E][2E]  */
  const float* ctx_b;   /* [E]      */
  const float* j_we;    /* [J][D]   */
  const float* j_wd;    /* [J][E]   */
  const float* j_b;     /* [J]      */
  const float* out_w;   /* [V][J]   */
  const float* out_b;   /* [V]      */
} rnntg_model_desc;

/* SearchParams (search.hpp:44-50).  max_symbols: 1..10 or
 * RNNTG_NO_SYMBOL_LIMIT (unlimited, at most 10 per frame as the reference's
 * safety cap; the frames stopped by it are counted in rnntg_stats).  With
 * S > 1 out_tokens must hold frame_splits[B] * min(S, 10) int32. */
typedef struct {
  int32_t beam_size;         /* >= 1 */
  int32_t max_symbols;       /* S: 1..10 or RNNTG_NO_SYMBOL_LIMIT */
  int32_t merge_op;          /* rnntg_merge_op */
  int32_t length_norm;       /* 0/1 */
  int32_t max_total_symbols; /* 0 = uncapped */
} rnntg_beam_params;

/* FsaSearchParams (fsa_search.hpp:33-37). */
typedef struct {
  double beam;          /* >= 0 */
  int32_t max_states;   /* >= 1 */
  int32_t max_contexts; /* >= 1 */
} rnntg_fsa_params;

/* Per-call counters (device-side, for the roofline and occupancy report). */
typedef struct {
  int64_t stream_frames;  /* sum over streams of frames decoded */
  int64_t joiner_rows;    /* joiner rows evaluated (distinct contexts) */
  int64_t arcs_expanded;  /* FSA: graph arcs expanded */
  int64_t lattice_arcs;   /* FSA: lattice arcs kept */
  int64_t tie_breaks;     /* exact-score ties resolved by the tie rules */
  int64_t kernel_launches;/* CUDA kernels launched by the call */
  float gpu_ms;           /* device time of the call (CUDA events) */
  float decode_ms;        /* device time of the persistent decode kernel */
  int64_t phase_cycles[4];/* beam kernel, summed over CTAs: h build, joiner
                             GEMM, row reduction, search step (SM cycles) */
  int64_t joiner_rows_computed; /* beam kernel: rows the GEMM tiles computed
                                   (row groups of 4, padding included) */
  int64_t gather_cycles;  /* beam kernel: cycles of the h build spent gathering
                             pe / pd rows (thread 0, summed over CTAs) */
  int64_t gemm_wait_cycles; /* beam kernel: joiner GEMM cycles thread 0 waited
                               for weight chunks (pipeline starvation) */
  int64_t capped_frames;  /* greedy_search with S unlimited: frames stopped by
                             the 10-symbol safety cap (search.hpp:31-34) */
} rnntg_stats;

const char* rnntg_last_error(void);
const char* rnntg_version(void);

rnntg_status rnntg_model_create(const rnntg_model_desc* desc, int32_t device,
                                rnntg_model_t* out);
rnntg_status rnntg_model_destroy(rnntg_model_t model);
/* Use `stream` (a cudaStream_t) for all work of this handle; NULL = the
 * handle's own (non-blocking) stream, which is NOT ordered with the legacy
 * default stream: a caller whose device inputs are produced on the legacy
 * default stream passes cudaStreamLegacy ((void*)0x1), not NULL.  Device
 * frames are read in stream order on the selected stream. */
rnntg_status rnntg_set_stream(rnntg_model_t model, void* stream);
rnntg_status rnntg_set_joiner_mode(rnntg_model_t model, int32_t mode);
rnntg_status rnntg_get_stats(rnntg_model_t model, rnntg_stats* out);

/*
 * Frames: `enc` is [frame_splits[B]][enc_dim] fp32, stream i owning rows
 * frame_splits[i] .. frame_splits[i+1]-1 (a ragged batch, like the
 * reference's std::vector<Mat<float>>).  frame_splits is always host memory.
 *
 * Results: ragged token lists.  out_splits[B+1] (host memory) receives the
 * prefix sums; out_tokens must hold frame_splits[B] int32 (S = 1 bounds each
 * stream by its frame count); out_scores (may be NULL) receives one fp64
 * score per stream.  `mem` says where enc / out_tokens / out_scores live.
 */
rnntg_status rnntg_greedy_search_batch(rnntg_model_t model, const float* enc,
                                       const int32_t* frame_splits, int32_t B,
                                       int32_t max_symbols, int32_t mem,
                                       int32_t* out_splits,
                                       int32_t* out_tokens);

/* greedy_search (search.hpp:76-100) for every stream of the batch: up to
 * max_symbols emissions per frame (RNNTG_NO_SYMBOL_LIMIT = unlimited, capped
 * at 10 per frame as the reference's kMaxSymbolsPerFrameSafety; the frames
 * that hit that cap are counted in *capped_frames, may be NULL).
 * out_tokens must hold frame_splits[B] * cap int32, cap = max_symbols, or 10
 * when unlimited. */
#define RNNTG_NO_SYMBOL_LIMIT 2147483647
rnntg_status rnntg_greedy_search(rnntg_model_t model, const float* enc,
                                 const int32_t* frame_splits, int32_t B,
                                 int32_t max_symbols, int32_t mem,
                                 int32_t* out_splits, int32_t* out_tokens,
                                 int64_t* capped_frames);

rnntg_status rnntg_beam_search_batch(rnntg_model_t model, const float* enc,
                                     const int32_t* frame_splits, int32_t B,
                                     const rnntg_beam_params* params,
                                     int32_t mem, int32_t* out_splits,
                                     int32_t* out_tokens, double* out_scores);

/* Decoding graph: CSR arcs grouped by source state (arcs of state s are
 * arc_splits[s] .. arc_splits[s+1]-1, in the order best-path tie rules see
 * them), natural-log fp64 weights.  Labels must be in [1, V) (graphs are
 * epsilon-free, fsa_search.hpp:103-111).  Host memory. */
rnntg_status rnntg_graph_create(rnntg_model_t model, int32_t num_states,
                                const int32_t* arc_splits, int32_t num_arcs,
                                const int32_t* dst, const int32_t* label,
                                const double* weight, rnntg_graph_t* out);
rnntg_status rnntg_graph_destroy(rnntg_graph_t graph);

/* One shared graph for all streams (the CLI decodes every utterance with the
 * same graph, rnnt_main.cpp:297).  out_scores = best_path score per stream,
 * -inf when the lattice has no complete path. */
rnntg_status rnntg_fsa_beam_search(rnntg_model_t model, const float* enc,
                                   const int32_t* frame_splits, int32_t B,
                                   rnntg_graph_t graph,
                                   const rnntg_fsa_params* params, int32_t mem,
                                   int32_t* out_splits, int32_t* out_tokens,
                                   double* out_scores);

/* Lattice of stream `stream` from the handle's last rnntg_fsa_beam_search
 * call, exactly as the reference's fsa_beam_search returns it
 * (fsa_search.hpp:301-317 build_lattice + make_fsa): nodes numbered frame by
 * frame in (context, state) order, arcs grouped by source node in generation
 * order, then one label-0 score-0 arc from every final-frame node into the
 * super-final node num_nodes-1 (final score 0).  Host arrays of `capacity`
 * entries; *num_arcs is always set (call with capacity 0 to size).  Returns
 * INVALID_ARGUMENT if capacity is too small. */
rnntg_status rnntg_fsa_lattice(rnntg_model_t model, int32_t stream,
                               int32_t* num_nodes, int32_t* num_arcs,
                               int32_t capacity, int32_t* src, int32_t* dst,
                               int32_t* label, double* score);

/* The Algorithm-1 step API (fsa_search.hpp:95-297; Algorithm 1):
 * the caller runs its own decoder + joiner between the context query and the
 * expansion, and hands in the log-prob rows -- expand_arcs' plug-in point
 * (fsa_search.hpp:59-61).  One open decode per model handle:
 *
 *   rnntg_fsa_stream_begin     init_streams (95-120) over B streams sharing
 *                              `graph` (which must outlive the decode, as
 *                              DecodeStream::graph; destroying it ends the
 *                              decode); num_frames[i] = frames stream i will
 *                              consume (the driver's DecodeStream::num_frames)
 *   rnntg_fsa_stream_contexts  get_contexts (124-154): per stream its distinct
 *                              active contexts in ascending packed order
 *                              (a*V + b); streams past their last frame (or
 *                              dead) contribute none.  out_row_splits [B+1]
 *                              is always written; contexts when capacity >=
 *                              out_row_splits[B] (call with 0 to size)
 *   rnntg_fsa_stream_step      expand_arcs (161-223) + prune_streams
 *                              (230-297) on the GPU with logprobs
 *                              [out_row_splits[B]][V] fp64 (host or device,
 *                              `mem`), row r = log p(. | context r); a step
 *                              without a fresh contexts call is the
 *                              reference's "stale get_contexts data"
 *                              (RNNTG_INTERNAL)
 *   rnntg_fsa_stream_end       finish_stream + lattice_to_best_seq(kMax) of
 *                              every stream: as rnntg_fsa_beam_search's
 *                              outputs; afterwards rnntg_fsa_lattice /
 *                              _text / _best read these lattices. */
rnntg_status rnntg_fsa_stream_begin(rnntg_model_t model, rnntg_graph_t graph,
                                    const rnntg_fsa_params* params, int32_t B,
                                    const int32_t* num_frames);
rnntg_status rnntg_fsa_stream_contexts(rnntg_model_t model,
                                       int32_t* out_row_splits,
                                       int32_t capacity, int32_t* out_contexts);
rnntg_status rnntg_fsa_stream_step(rnntg_model_t model, const double* logprobs,
                                   int32_t mem);
rnntg_status rnntg_fsa_stream_end(rnntg_model_t model, int32_t* out_splits,
                                  int32_t* out_tokens, double* out_scores);

/* lattice_to_best_seq(lattice, kLogAdd, nbest_n, seed) (fsa_search.hpp:
 * 410-425) for every stream of the last rnntg_fsa_beam_search, on the GPU:
 * n-best sampling with DetRng(seed) (fsa.hpp:390-448), blank-free
 * deduplication (452-463), per-sequence total log-probability (533-540),
 * argmax with the reference's tie rule.  Same results as the reference
 * function on the same lattices (the CLI's `--merge log_add` decode,
 * rnnt_main.cpp:302).  merge_op must be RNNTG_MERGE_LOG_ADD (kMax is the
 * search's own output).  Host outputs: out_splits [B+1], out_tokens (<= sum
 * T), out_logprob [B] (may be NULL): the winner's total, -inf if the
 * lattice has no complete path (empty sequence). */
rnntg_status rnntg_fsa_lattice_best(rnntg_model_t model, int32_t merge_op,
                                    int32_t nbest_n, uint64_t seed,
                                    int32_t* out_splits, int32_t* out_tokens,
                                    double* out_logprob);

/* The lattice of `stream` as text, byte-identical to the reference's
 * serialize_fsa_text (fsa.hpp:243-262) of that stream's fsa_beam_search
 * lattice, prefixed with serialize_lattice's "# stream=S frames=T" line
 * (fsa_search.hpp:429-435) when with_header != 0 -- the CLI's
 * lattice_NNNN.txt (rnnt_main.cpp:303-307).  *length is always set (bytes,
 * excluding the terminating NUL); call with capacity 0 to size, then with
 * capacity >= *length + 1. */
rnntg_status rnntg_fsa_lattice_text(rnntg_model_t model, int32_t stream,
                                    int32_t with_header, char* buf,
                                    int64_t capacity, int64_t* length);

/* The reference's toy encoder on the GPU (encoder_forward, model.hpp:224-238;
 * SURVEY.md §8f "next" row 3): enc[t] = tanhf(b2 + W2 . tanhf(b1 + W1 . f[t])),
 * bit-exact with the reference (same sequential fp32 affine and glibc tanhf
 * as the joiner).  Weights are fp32 row-major host arrays in param_views
 * naming; enc_dim must equal the model's enc_dim. */
typedef struct {
  int32_t feat_dim;      /* F */
  const float* enc_w1;   /* [D][F] */
  const float* enc_b1;   /* [D]    */
  const float* enc_w2;   /* [D][D] */
  const float* enc_b2;   /* [D]    */
} rnntg_encoder_desc;

/* Page-locked (pinned) host memory for staging inputs and outputs: a copy
 * from it is one DMA at full PCIe / C2C speed and stays asynchronous
 * (cudaHostAlloc, portable).  No reference counterpart: the C++ drop-in
 * (rnnt_gpu.hpp) gathers a batch's features into one such buffer per
 * Context instead of a fresh pageable vector per call. */
rnntg_status rnntg_host_alloc(size_t bytes, void** out);
rnntg_status rnntg_host_free(void* ptr);

rnntg_status rnntg_model_set_encoder(rnntg_model_t model,
                                     const rnntg_encoder_desc* desc);
/* feats: [frame_splits[B]][F]; enc_out: [frame_splits[B]][D].  `mem` says
 * where feats and enc_out live (host or this model's device). */
rnntg_status rnntg_encoder_forward(rnntg_model_t model, const float* feats,
                                   const int32_t* frame_splits, int32_t B,
                                   int32_t mem, float* enc_out);

/* Synthetic inputs bit-identical to the reference's (host only, no GPU).
 *
 * rnntg_init_model_weights <- init_model (model.hpp:129-169): DetRng(seed)
 *   uniform(-1/sqrt(fan_in), 1/sqrt(fan_in)) fills in the reference's order
 *   (common.hpp:86-105, model.hpp:94-97).  Every pointer of `w` receives its
 *   param_views-shaped array (row-major fp32); a NULL pointer skips the
 *   array but keeps the draw order.  The reference's ModelConfig seed.
 * rnntg_gaussian_features  <- SURVEY.md §8(d) synthetic features: stream i of
 *   B gets T x feat_dim floats (float)DetRng(seed0 + i).gaussian()
 *   (Box-Muller with spare, common.hpp:108-121), stored [B][T][feat_dim].
 *   threads <= 0: all hardware threads. */
typedef struct {
  int32_t vocab_size, feat_dim, enc_dim, emb_dim, joiner_dim;
  uint64_t seed;
} rnntg_model_config;

typedef struct {
  float *enc_w1, *enc_b1, *enc_w2, *enc_b2;
  float *emb, *ctx_w, *ctx_b, *j_we, *j_wd, *j_b, *out_w, *out_b;
} rnntg_weight_ptrs;

rnntg_status rnntg_init_model_weights(const rnntg_model_config* cfg,
                                      const rnntg_weight_ptrs* w);
rnntg_status rnntg_gaussian_features(uint64_t seed0, int32_t B, int32_t T,
                                     int32_t feat_dim, int32_t threads,
                                     float* out);

/* Kernel-level entry points (bit-exactness tests of the joiner pieces).
 * All pointers are host memory. */
rnntg_status rnntg_debug_decoder_projection(rnntg_model_t model,
                                            const int32_t* contexts, int32_t n,
                                            float* pd_out);
rnntg_status rnntg_debug_joiner_logits(rnntg_model_t model, const float* enc,
                                       const int32_t* contexts, int32_t n,
                                       float* logits_out);
/* tanhf port over x[i], i < n (exhaustive sweep support): writes a 64-bit
 * FNV-style hash of the output bits of every 2^24-input chunk starting at
 * chunk `first_chunk` into hashes[0..num_chunks). */
rnntg_status rnntg_debug_tanhf_chunk_hashes(int32_t device, int32_t first_chunk,
                                            int32_t num_chunks,
                                            uint64_t* hashes);

/* The decoders' log-softmax normaliser over n rows of V fp32 logits:
 * lse[r] = double(max) + log(sum_k exp(double(l_k) - max)), the reference's
 * detail::log_softmax_row (model.hpp:115-125) bit for bit. */
rnntg_status rnntg_debug_log_softmax_lse(int32_t device, const float* logits,
                                         int32_t n, int32_t V, double* lse);
/* The device ports of glibc's exp (op 0), log (1), log1p (2) and the
 * decoders' branch-light exp (3) over x[0..n). */
rnntg_status rnntg_debug_f64_math(int32_t device, int32_t op, const double* x,
                                  int64_t n, double* y);

#ifdef __cplusplus
}
#endif

#endif /* RNNTG_H_ */
