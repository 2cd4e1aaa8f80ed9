/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of FlexCTC's batched CTC beam search
 * (§III-C, Algorithm 1), its NGPU-LM shallow fusion term (P:92, P:129,
 * P:143) evaluated by the direct ARPA backoff recursion, and its GPU-PB phrase-boosting
 * term evaluated by naive suffix matching (no failure automaton).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library. It shares no code, header, table or constant generator with the CUDA
 * product under paper_2508_07315_b200/ and never imports it.
 *
 * Precision: the paper measured in float32 ("using float32 arithmetic"), so the parity
 * oracle computes in fp32 with the canonical operation order of DESIGN.md reading R19. An fp64
 * instantiation of the same template serves the exactness pins (brute force, CTC forward).
 */
#ifndef FLEXCTC_ORACLE_H
#define FLEXCTC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t beam;          /* K */
    double alpha_lm;       /* α_LM of Eq. (1) */
    double alpha_bt;       /* α_BT of Eq. (1) */
    double beta;           /* β, added to non-blank non-repeat candidates (Alg. 1) */
    double theta;          /* θ-prune (Alg. 1); +inf disables */
    int32_t merge_mode;    /* 0 = log-sum-exp, 1 = max (R13) */
    int32_t retract_boost_at_eos; /* DESIGN.md R17; default 0 */
    int32_t fuse_repeats;  /* 1: repeat candidates also get the LM / BT terms (PAPER.md P:167 variant) */
    int32_t merge_first;   /* 1: recombine duplicate (prefix, last) candidates BEFORE the TopK (reading R27) */
} oracle_cfg;

const char* oracle_last_error(void);

/* ---- LM: ARPA text -> direct backoff evaluator (R7) ---- */
void* oracle_lm_load(const char* arpa_path, int32_t vocab_size, const char* const* token_symbols);
void  oracle_lm_free(void* lm);
int32_t oracle_lm_order(const void* lm);
/* log P(w | <s> hist[0..n)) in nats; w = decoder token, or -1 for </s>. f32 != 0 -> fp32 path. */
double oracle_lm_logp(const void* lm, const int32_t* hist, int32_t n, int32_t w, int32_t f32);
/* the same for m tokens after one history: out[i] = log P(ws[i] | hist) */
void oracle_lm_logp_many(const void* lm, const int32_t* hist, int32_t n, const int32_t* ws, int32_t m, int32_t f32,
                         double* out);
/* Σ_i log P(tok_i | <s> tok_<i) + log P(</s> | <s> tok), fp64 */
double oracle_lm_seq(const void* lm, const int32_t* toks, int32_t n);

/* ---- Boosting: phrase set -> naive suffix matcher (R17) ---- */
void* oracle_boost_build(const int32_t* tokens, const int64_t* offsets, int32_t n_phrases,
                         double token_weight, int32_t vocab_size);
void  oracle_boost_free(void* bt);
/* delta(prefix, w) = dC(v) + U(v) - U(u) with u = state(prefix), v = state(prefix + w) */
double oracle_boost_delta(const void* bt, const int32_t* prefix, int32_t n, int32_t w, int32_t f32);
double oracle_boost_U(const void* bt, const int32_t* prefix, int32_t n, int32_t f32);
/* length of state(prefix) (longest suffix of prefix that is a phrase prefix) */
int32_t oracle_boost_state_depth(const void* bt, const int32_t* prefix, int32_t n);

/* ---- Decoding (Alg. 1), fp32, utterance-parallel over nthreads ----
 * log_probs[b*stride_b + t*stride_t + w], blank = Vp1-1. Outputs as the product's C ABI:
 * tokens/timestamps/alignment [B,T] (-1 padded), num_tokens [B], scores [B]. */
int32_t oracle_decode_f32(const float* log_probs, int64_t stride_b, int64_t stride_t,
                          const int32_t* lengths, int32_t B, int32_t T, int32_t Vp1,
                          const oracle_cfg* cfg, const void* lm, const void* bt, int32_t nthreads,
                          int32_t* out_tokens, int32_t* out_num_tokens, float* out_scores,
                          int32_t* out_timestamps, int32_t* out_alignment);

/* One utterance in fp64 (or fp32 if f32), returning every final merged hypothesis
 * (n-best, sorted by score desc, slot asc). tokens_out is [max_out, T]. Returns count. */
int32_t oracle_decode_nbest(const double* log_probs, int32_t T, int32_t Vp1, int32_t L,
                            const oracle_cfg* cfg, const void* lm, const void* bt, int32_t f32,
                            int32_t max_out, int32_t* tokens_out, int32_t* lens_out,
                            double* scores_out);

/* ---- input side (reading R25): log-softmax of bf16 logits ----
 * Row i of n_rows holds Vp1 bf16 logits at x + i*stride (elements). With the logits as exact
 * reals: m = max_w x_w; S = sum_w exp(x_w - m) in fp64, index order; lse = m + log(S) (fp64);
 * out[i*Vp1 + w] = (float)(x_w - lse), the fp64 difference rounded once. Returns 0. */
int32_t oracle_log_softmax_bf16(const uint16_t* x, int64_t n_rows, int64_t stride, int32_t Vp1, float* out);

#ifdef __cplusplus
}
#endif
#endif
