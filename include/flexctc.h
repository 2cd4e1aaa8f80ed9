/* flexctc.h — C ABI of the B200-native FlexCTC hot path (libflexctc.so).
 *
 * What it computes: batched CTC beam search with n-gram LM shallow fusion and phrase boosting,
 * PAPER.md §III-C Algorithm 1 with the score of Eq. (1):
 *     s = log P_CTC + α_LM·log P_LM + α_BT·log P_PB + β·N
 * The readings of the garbled / silent passages (blank id, merge key, combiner, tie rule, ...)
 * are listed in DESIGN.md ("Readings R1-R23"); each is cited below where it decides behaviour.
 *
 * Conventions
 *  - Handles are immutable after creation and may be shared across threads and streams of the
 *    device they were created for. The library owns them; *_free releases them.
 *  - Every input, output and workspace buffer is owned by the caller.
 *  - flexctc_decode only enqueues work on `stream` (one length-sort kernel + one persistent
 *    beam kernel) and never synchronises. Host-side validation errors are returned before any
 *    launch. Device-side anomalies (length > T, length < 0) are clamped and flagged in the
 *    workspace; read them with flexctc_check after the stream has synchronised.
 *  - Passing host memory to flexctc_decode returns FLEXCTC_ERR_INVALID_ARG: there is no CPU
 *    path. flexctc_decode_host is the end-to-end entry for host buffers (it copies to the
 *    device, decodes on the GPU, copies back and synchronises).
 *  - All status-returning functions set a thread-local message readable with
 *    flexctc_last_error().
 */
#ifndef FLEXCTC_H
#define FLEXCTC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct flexctc_lm flexctc_lm;       /* n-gram LM in the sorted-arc state layout */
typedef struct flexctc_boost flexctc_boost; /* Aho-Corasick boosting automaton        */
typedef struct CUstream_st* flexctc_stream; /* == cudaStream_t (NULL = legacy default) */

typedef enum {
    FLEXCTC_OK = 0,
    FLEXCTC_ERR_INVALID_ARG = 1,  /* shapes, ranges, host pointers, wrong device */
    FLEXCTC_ERR_PARSE = 2,        /* malformed ARPA (message has file:line), missing </s> */
    FLEXCTC_ERR_VOCAB_BIND = 3,   /* decoder token absent from the LM and no <unk> */
    FLEXCTC_ERR_CAPACITY = 4,     /* V+1 or K beyond the kernel's limits, workspace too small */
    FLEXCTC_ERR_CUDA = 5,         /* a CUDA runtime call failed (message has the CUDA error) */
    FLEXCTC_ERR_OOM = 6,          /* device or host allocation failed */
    FLEXCTC_ERR_IO = 7            /* cannot open / read a file */
} flexctc_status;

/* Device-side flags reported by flexctc_check (bitwise OR). */
#define FLEXCTC_FLAG_LENGTH_CLAMPED_HIGH 1u /* some lengths[b] > T: clamped to T  */
#define FLEXCTC_FLAG_LENGTH_CLAMPED_LOW 2u  /* some lengths[b] < 0: clamped to 0  */
#define FLEXCTC_FLAG_STREAM_TIMEOUT 4u      /* flexctc_decode_host: a frame chunk never arrived
                                               (10 s watchdog); the outputs are invalid        */

const char* flexctc_last_error(void);
const char* flexctc_version(void);

/* ---------------------------------------------------------------------------------------
 * NGPU-LM replacement (§II-D, §III-B; Alg. 1 P:114-116, P:128-129,
 * P:142-143).
 *
 * Parses an ARPA file (log10 values converted to nats once: (float)(log10 · ln 10), reading R7)
 * and builds the device layout: states = listed contexts (length <= order-1), per-state arcs
 * sorted by decoder token (CSR), backoff state + weight per state, dense root row, and per
 * state the precomputed EOS score LM.Final (R19: fp32, same accumulation order as the oracle).
 *   vocab_size     V, the number of non-blank decoder tokens; decoder token i is the LM
 *                  symbol token_symbols[i] (or the decimal string "i" when token_symbols is
 *                  NULL). A symbol missing from the LM maps to <unk>, else
 *                  FLEXCTC_ERR_VOCAB_BIND.
 *   device         CUDA device ordinal that receives the arrays, or -1 for a host-only handle
 *                  (usable by the *_host_* inspection calls and by nothing else).
 * Errors: FLEXCTC_ERR_IO, FLEXCTC_ERR_PARSE (count mismatch, unknown symbol in an n-gram,
 * missing \end\ or </s>), FLEXCTC_ERR_VOCAB_BIND, FLEXCTC_ERR_CUDA/OOM. *out is NULL on error.
 * ------------------------------------------------------------------------------------- */
flexctc_status flexctc_lm_load(const char* arpa_path, int32_t vocab_size,
                               const char* const* token_symbols, int32_t device,
                               flexctc_lm** out);
void flexctc_lm_free(flexctc_lm* lm);

typedef struct {
    int32_t order, vocab_size, n_states, start_state;
    int64_t n_arcs;
    int64_t device_bytes;
} flexctc_lm_info;
flexctc_status flexctc_lm_get_info(const flexctc_lm* lm, flexctc_lm_info* info);

/* Host-side query on the built layout (test/inspection; no GPU needed):
 * log P(token | state) in nats and the next state (token = -1 queries </s>, next = state). */
flexctc_status flexctc_lm_host_query(const flexctc_lm* lm, int32_t state, int32_t token,
                                     float* logp, int32_t* next_state);

/* Batch form: n (state, token) pairs from host arrays; logp[i], next_state[i] written (host).
 * FLEXCTC_ERR_INVALID_ARG on a NULL array or any state/token out of range (outputs undefined). */
flexctc_status flexctc_lm_host_query_batch(const flexctc_lm* lm, int64_t n, const int32_t* states,
                                           const int32_t* tokens, float* logp, int32_t* next_state);

/* The pre-prune bound the kernels use for a state (test/inspection): *ub >= max over decoder
 * tokens w of log P(w | state) (nats; rounded up by a relative 1e-5 margin), *eos = LM.Final. */
flexctc_status flexctc_lm_host_bound(const flexctc_lm* lm, int32_t state, float* ub, float* eos);

/* ---------------------------------------------------------------------------------------
 * GPU-PB replacement (§III-B P:92 "phrase prefix tree ... Aho-Corasick ... boosting
 * scores along the prefix tree based on node depth"; Alg. 1).
 * Reward law (reading R17): C(n) = w·depth(n); committed(n) = C(deepest final
 * ancestor-or-self); U = C - committed; pcom = C(deepest final strict ancestor);
 * delta(u, a) = [v final]·(C(v) - pcom(v)) + U(v) - U(u) with v the Aho-Corasick transition.
 *   tokens/offsets  CSR phrase list in host memory: phrase i = tokens[offsets[i] .. offsets[i+1]).
 *   token_weight    w (> 0), nats per matched token; the decoder scales it by α_BT.
 * The device layout is the full transition table [nodes × V] of (next node, delta), plus U
 * and max-delta per node. Errors: FLEXCTC_ERR_INVALID_ARG (empty list, empty phrase, token
 * outside [0, V), w <= 0), FLEXCTC_ERR_CAPACITY (table > 2^31 entries), CUDA/OOM.
 * ------------------------------------------------------------------------------------- */
flexctc_status flexctc_boost_build(const int32_t* tokens, const int64_t* offsets,
                                   int32_t n_phrases, float token_weight, int32_t vocab_size,
                                   int32_t device, flexctc_boost** out);
void flexctc_boost_free(flexctc_boost* boost);
flexctc_status flexctc_boost_host_query(const flexctc_boost* boost, int32_t node, int32_t token,
                                        float* delta, int32_t* next_node, float* U_node);
flexctc_status flexctc_boost_num_nodes(const flexctc_boost* boost, int32_t* n_nodes);

/* Batch form of flexctc_boost_host_query over n (node, token) pairs (host arrays). */
flexctc_status flexctc_boost_host_query_batch(const flexctc_boost* boost, int64_t n, const int32_t* nodes,
                                              const int32_t* tokens, float* delta, int32_t* next_node);

/* Exception signature of a node (test/inspection): bit (token · 0x9E3779B1 mod 2^32) >> 26 is
 * set for every token whose transition from `node` differs from the root's. For any other token
 * δ(node, a) = δ(root, a) and delta(node, a) = fl(delta(root, a) - U(node)) exactly, which lets the
 * kernels serve it from the root row. The root's signature is 0. */
flexctc_status flexctc_boost_host_signature(const flexctc_boost* boost, int32_t node, uint64_t* sig);

/* ---------------------------------------------------------------------------------------
 * Decoding configuration (Eq. (1) weights P:96-98, θ P:237).
 * ------------------------------------------------------------------------------------- */
typedef struct {
    int32_t beam;                 /* K, 1..256 */
    float alpha_lm;               /* α_LM (used iff lm != NULL) */
    float alpha_bt;               /* α_BT (used iff boost != NULL) */
    float beta;                   /* β, added to non-blank non-repeat candidates (R8) */
    float theta;                  /* θ-prune; +INFINITY disables pruning (R10) */
    int32_t merge_mode;           /* 0 = log-sum-exp (default), 1 = max (R13) */
    int32_t retract_boost_at_eos; /* 1: score -= α_BT·U(state) at EOS (R17); default 0 */
    int32_t fuse_repeats;         /* 1: repeat candidates (w == last label) also get the α_LM / α_BT
                                     terms, at every occurrence (the variant the
                                     authors tried; no β, no state advance); default 0 = Alg. 1 */
    int32_t merge_first;          /* 1: recombine duplicate (transcript, last label) candidates BEFORE
                                     the TopK (BJ north_star "merges duplicate prefixes ..., selects
                                     the top-K"; reading R27): groups ranked by merged
                                     score, flat index of the best member on ties; θ-prune against the
                                     best group. Runs merge_first_kernel (1-best only: nbest must be
                                     1). Default 0 = Alg. 1's TopK -> recombine order */
} flexctc_config;

/* Workspace bytes for a decode of B utterances of up to T frames with V+1 = Vp1 tokens.
 * Holds the backpointers (B·T·K·3 bytes: u8 parent + u16 label, "token and
 * pointer tensors"), chunk ancestors, the LPT order and the device flags. */
size_t flexctc_workspace_bytes(int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg);

/* ---------------------------------------------------------------------------------------
 * flexctc_decode — Algorithm 1 for a batch, 1-best output (R22).
 * K = 1 runs the greedy kernels (one bandwidth-bound frame-summary pass
 * over D, then a warp per utterance; same outputs as Algorithm 1 with a beam of one).
 *   log_probs   device fp32, element (b, t, w) at log_probs[b·stride_b + t·stride_t + w];
 *               unit stride over w; blank id = Vp1-1 (R1). Frames t >= lengths[b] are never
 *               read (R16: NaN padding is allowed).
 *   lengths     device int32 [B]; values outside [0, T] are clamped and flagged.
 *   B, T, Vp1   batch, padded frames, V+1 (2 <= Vp1 <= 8192). With T = 0 the [B, T] arrays
 *               (log_probs, out_tokens, out_timestamps, out_alignment) may be NULL.
 *   cfg         host pointer; lm / boost may be NULL (fusion term off).
 *   workspace   device buffer of at least flexctc_workspace_bytes(B, T, Vp1, cfg) bytes.
 *   out_tokens      device int32 [B, T]: best transcript, -1 padded.
 *   out_num_tokens  device int32 [B].
 *   out_scores      device fp32 [B]: Eq. (1) total incl. the EOS term, merged (R15).
 *   out_timestamps  device int32 [B, T] or NULL: frame of each token's emission (R20), -1 pad.
 *   out_alignment   device int32 [B, T] or NULL: frame labels of the best path, -1 pad.
 * Returns FLEXCTC_ERR_INVALID_ARG for bad shapes/config or host pointers, ERR_CAPACITY for
 * Vp1 / K beyond the limits or a short workspace, ERR_CUDA for launch failures.
 * ------------------------------------------------------------------------------------- */
flexctc_status flexctc_decode(const float* log_probs, int64_t stride_b, int64_t stride_t,
                              const int32_t* lengths, int32_t B, int32_t T, int32_t Vp1,
                              const flexctc_config* cfg, const flexctc_lm* lm,
                              const flexctc_boost* boost, void* workspace,
                              size_t workspace_bytes, flexctc_stream stream,
                              int32_t* out_tokens, int32_t* out_num_tokens, float* out_scores,
                              int32_t* out_timestamps, int32_t* out_alignment);

/* ---------------------------------------------------------------------------------------
 * flexctc_decode_nbest — flexctc_decode returning the `nbest` best final hypotheses per
 * utterance instead of one (SPEC --nbest S:494; the final merge R15 ranks
 * the merged hypotheses by (score desc, slot asc), rank 0 is flexctc_decode's output).
 *   nbest           1 <= nbest <= cfg->beam (else FLEXCTC_ERR_INVALID_ARG).
 *   out_tokens      device int32 [B, nbest, T], -1 padded; rows past the number of surviving
 *                   hypotheses are empty.
 *   out_num_tokens  device int32 [B, nbest] (0 for empty rows).
 *   out_scores      device fp32 [B, nbest] (-inf for empty rows).
 *   out_timestamps  device int32 [B, nbest, T] or NULL.
 * Everything else (arguments, workspace, errors, asynchrony) as flexctc_decode.
 * ------------------------------------------------------------------------------------- */
flexctc_status flexctc_decode_nbest(const float* log_probs, int64_t stride_b, int64_t stride_t,
                                    const int32_t* lengths, int32_t B, int32_t T, int32_t Vp1,
                                    const flexctc_config* cfg, const flexctc_lm* lm,
                                    const flexctc_boost* boost, void* workspace,
                                    size_t workspace_bytes, flexctc_stream stream, int32_t nbest,
                                    int32_t* out_tokens, int32_t* out_num_tokens, float* out_scores,
                                    int32_t* out_timestamps);

/* ---------------------------------------------------------------------------------------
 * flexctc_decode_logits_bf16 — flexctc_decode over bf16 LOGITS instead of fp32 log-probs
 * (the log-softmax the acoustic model would otherwise run, moved into the
 * decoder's input side; the bf16 input halves the bytes read from HBM and copied from the host).
 * One bandwidth-bound pass normalises every frame t < lengths[b] (reading R25: m = max,
 * S = sum exp(x - m) and lse = m + log S in fp64, D = (float)(x - lse)) into the workspace, then
 * the decode runs on D exactly as flexctc_decode.
 *   logits      device bf16 bit patterns (uint16), element (b, t, w) at
 *               logits[b·stride_b + t·stride_t + w]; unit stride over w; NULL allowed iff T = 0.
 *   workspace   at least flexctc_logits_workspace_bytes(B, T, Vp1, cfg) bytes (the decode's
 *               workspace plus the dense fp32 [B, T, Vp1] log-probs).
 * Everything else (arguments, outputs, errors, asynchrony) as flexctc_decode.
 * ------------------------------------------------------------------------------------- */
size_t flexctc_logits_workspace_bytes(int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg);
flexctc_status flexctc_decode_logits_bf16(const uint16_t* logits, int64_t stride_b, int64_t stride_t,
                                          const int32_t* lengths, int32_t B, int32_t T, int32_t Vp1,
                                          const flexctc_config* cfg, const flexctc_lm* lm,
                                          const flexctc_boost* boost, void* workspace,
                                          size_t workspace_bytes, flexctc_stream stream,
                                          int32_t* out_tokens, int32_t* out_num_tokens,
                                          float* out_scores, int32_t* out_timestamps,
                                          int32_t* out_alignment);

/* Measurement hook: when both are non-NULL, subsequent flexctc_decode calls on this thread
 * record `ev_start` (a cudaEvent_t) immediately before and `ev_stop` immediately after the
 * persistent beam kernel on the decode stream, so callers can time that kernel alone.
 * Pass NULL, NULL to disable. */
void flexctc_set_profile_events(void* ev_start, void* ev_stop);

/* Measurement hook per stage of the decode: stage 0 is the beam kernel (the same as
 * flexctc_set_profile_events), stage 1 the frame compaction pass (the bandwidth-bound pass over
 * every valid frame row; only decodes that take the warp path, 2 <= K <= 32,
 * launch it). Events are cudaEvent_t, recorded on the decode stream immediately before and after
 * the stage's kernel; NULL, NULL disables the stage. Returns FLEXCTC_ERR_INVALID_ARG for an
 * unknown stage. */
flexctc_status flexctc_set_stage_events(int32_t stage, void* ev_start, void* ev_stop);

/* Name of the main (frame-loop) kernel the last decode on this thread launched, e.g.
 * "warp_beam_kernel+helpers", "warp_beam_kernel", "ctc_beam_kernel", "greedy_fused_kernel",
 * "greedy_chain_kernel" (static string, never NULL; "" before the first decode). */
const char* flexctc_last_kernel(void);

/* Device counters of the last decode that used `workspace` (call after the stream has
 * synchronised); copies min(n, 48) u64 values: frames, sum of live slots, sum of listed tokens,
 * sparse exact evaluations, dense frames, LM rows built, dense exact evaluations, buffer
 * compactions, top-token stages, deferred next-state queries, then SM cycles (summed over CTAs,
 * thread 0) of frame phases 1-3, 4, LM row builds, 5, 6-7, the count of frames with listed
 * tokens and their cycles, finer phase cycles (timers builds), and at word 35 the frames the CTA
 * kernel's settled-beam fast path took. The warp kernel reuses words 21-29 for its own counters. */
flexctc_status flexctc_get_stats(const void* workspace, uint64_t* out, int32_t n);

/* Reads the device flags of the last decode that used `workspace` (call after the stream has
 * synchronised). */
flexctc_status flexctc_check(const void* workspace, uint32_t* device_flags);

/* End-to-end entry for HOST buffers: copies log_probs [B, T, Vp1] (dense, stride Vp1) and
 * lengths to the device (into `device_scratch`, which must hold
 * flexctc_host_scratch_bytes(B, T, Vp1, cfg) bytes of device memory), decodes, copies the
 * outputs back into host arrays and synchronises `stream`. Pinned host memory makes the
 * copies asynchronous DMA. Outputs as flexctc_decode, in host memory.
 * For K > 1 the input is streamed: the beam kernel is launched first and frame chunks
 * [t0, t1) of every utterance (only frames t < lengths[b]) are copied on a library-owned copy
 * stream, each followed by a "frames ready" word the row loaders wait on, so the copy overlaps
 * the frame recurrence (flexctc_host_streaming() says whether this is active). The host
 * buffers must stay unchanged until the call returns. A chunk that never lands (a failed copy)
 * releases the kernel after 10 s: the call then returns FLEXCTC_ERR_CUDA.
 *   out_flags   host uint32 or NULL: the device flags of this decode (FLEXCTC_FLAG_*: length
 *               clamps, stream timeout), read after the final synchronisation. */
size_t flexctc_host_scratch_bytes(int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg);
/* 1 if flexctc_decode_host on the current device streams its input (frame chunks copied on a
 * library-owned copy stream while the beam kernel runs, each chunk signalled by a stream memory
 * operation), 0 if it copies everything before decoding (K = 1, no stream memory operations,
 * or the FLEXCTC_NO_STREAM_INPUT environment switch). */
int32_t flexctc_host_streaming(void);
flexctc_status flexctc_decode_host(const float* log_probs_host, const int32_t* lengths_host,
                                   int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg,
                                   const flexctc_lm* lm, const flexctc_boost* boost,
                                   void* device_scratch, size_t scratch_bytes,
                                   flexctc_stream stream, int32_t* out_tokens,
                                   int32_t* out_num_tokens, float* out_scores,
                                   int32_t* out_timestamps, uint32_t* out_flags);

/* flexctc_decode_host over bf16 LOGITS (uint16 bit patterns, dense [B, T, Vp1] host buffer):
 * the end-to-end entry of the bf16 input side. The H2D transfer is
 * 2 B per logit; on the device every frame t < lengths[b] is normalised exactly as
 * flexctc_decode_logits_bf16 does (reading R25) into an fp32 log-prob buffer in the scratch, then
 * decoded as flexctc_decode_host. With K > 1 and B < #SMs the copy is streamed in frame chunks
 * and each chunk is normalised on the copy stream before its "frames ready" signal, so the
 * transfer and the normalisation overlap the frame recurrence. device_scratch: at least
 * flexctc_host_scratch_bytes_bf16(B, T, Vp1, cfg) bytes of device memory. Everything else
 * (outputs, flags, errors, synchronisation) as flexctc_decode_host. */
size_t flexctc_host_scratch_bytes_bf16(int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg);
flexctc_status flexctc_decode_host_bf16(const uint16_t* logits_host, const int32_t* lengths_host,
                                        int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg,
                                        const flexctc_lm* lm, const flexctc_boost* boost,
                                        void* device_scratch, size_t scratch_bytes,
                                        flexctc_stream stream, int32_t* out_tokens,
                                        int32_t* out_num_tokens, float* out_scores,
                                        int32_t* out_timestamps, uint32_t* out_flags);

#ifdef __cplusplus
}
#endif
#endif /* FLEXCTC_H */
