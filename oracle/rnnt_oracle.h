/* CPU restatement of the reference's one-symbol-per-frame decoding path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path in
 * paper_2211_00484_b200/ and may be called only from tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg.  It is never
 * linked into, loaded by, or used as a fallback for the product library.
 *
 * It restates the reference (rnnt-kit, /root/reference/proj/include/rnnt)
 * function by function; each function in rnnt_oracle.cpp cites the
 * reference file:line it follows.  Unlike the reference it takes encoder
 * frames directly (the north-star input) and also returns the winning beam
 * score, which the reference's beam_search computes but does not return
 * (search.hpp:261-276).  Parity of this restatement with the compiled
 * reference (oracle/_ref/librnnt_ref.so) is pinned in
 * tests/test_oracle_vs_reference.py; its known-answer checks against the
 * reference's own unit-test fixtures live in tests/test_oracle_kats.py.
 */
#ifndef RNNT_ORACLE_H_
#define RNNT_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Weights in the reference's param_views naming (model.hpp:75-82), fp32,
 * row-major:  emb[V][E], ctx_w[E][2E], ctx_b[E], j_we[J][D], j_wd[J][E],
 * j_b[J], out_w[V][J], out_b[V]. */
typedef struct {
  int32_t V, D, E, J;
  const float *emb, *ctx_w, *ctx_b, *j_we, *j_wd, *j_b, *out_w, *out_b;
} orc_model;

/* Decoding graph in CSR form (fsa.hpp:54-80): arcs of state s are
 * [arc_splits[s], arc_splits[s+1]); weights are natural-log doubles. */
typedef struct {
  int32_t num_states, num_arcs;
  const int32_t *arc_splits, *dst, *label;
  const double* weight;
} orc_graph;

/* Lattice arcs of one stream, in the reference's make_fsa order (stable by
 * src, generation order within src), plus the super-final hop arcs. */
typedef struct {
  int32_t num_nodes; /* including the super-final node */
  int32_t num_arcs;
  int32_t *src, *dst, *label;
  double* score;
} orc_lattice;

float orc_tanhf(float x);
/* y[m][n] = (bias ? bias[n] : 0) + sum_k w[n][k]*x[m][k], sequential fp32. */
void orc_affine(const float* w, const float* bias, const float* x, int32_t M,
                int32_t N, int32_t K, float* y);
void orc_encoder(const float* w1, const float* b1, const float* w2,
                 const float* b2, int32_t F, int32_t D, const float* feats,
                 int32_t T, float* enc);
void orc_decoder_project(const orc_model* m, const int32_t* ctxs, int32_t n,
                         float* pd);
void orc_joiner_logits_from_proj(const orc_model* m, const float* pe,
                                 const float* pd, float* logits);
void orc_log_softmax(const float* logits, int32_t n, double* out);

int orc_greedy_batch(const orc_model* m, const float* enc,
                     const int32_t* frame_splits, int32_t B, int threads,
                     int32_t* out_splits, int32_t* out_tokens);

int orc_beam_search(const orc_model* m, const float* enc,
                    const int32_t* frame_splits, int32_t B, int32_t beam_size,
                    int32_t merge_op, int32_t length_norm,
                    int32_t max_total_symbols, int threads,
                    int32_t* out_splits, int32_t* out_tokens,
                    double* out_scores);

/* lattices: optional array of B orc_lattice; arrays are malloc'd by the
 * oracle and released with orc_lattice_free. */
int orc_fsa_beam_search(const orc_model* m, const float* enc,
                        const int32_t* frame_splits, int32_t B,
                        const orc_graph* g, double beam, int32_t max_states,
                        int32_t max_contexts, int threads, int32_t* out_splits,
                        int32_t* out_tokens, double* out_scores,
                        orc_lattice* lattices);
void orc_lattice_free(orc_lattice* l);

void orc_tanhf_chunk_hashes(int32_t first_chunk, int32_t num_chunks,
                            int threads, uint64_t* out);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* RNNT_ORACLE_H_ */
