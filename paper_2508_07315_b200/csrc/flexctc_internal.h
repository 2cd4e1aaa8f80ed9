// Internal definitions of libflexctc (product code; never shared with oracle/).
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <vector_types.h>

#include "../../include/flexctc.h"

namespace flexctc {

void set_error(const std::string& msg);
// name of the main kernel the last decode on this thread launched (flexctc_last_kernel)
void set_kernel_name(const char* name);
flexctc_status fail(flexctc_status st, const std::string& msg);

// ---------------------------------------------------------------------------------------
// LM device layout ("sorted-arc, state-indexed"; DESIGN.md §Data layout)
//   state header  int4 {arc_off, arc_deg, backoff_state, backoff_weight(f32 bits)}
//   arcs          arc_tok u16 (decoder token, sorted within a state) + arc_val {f32 logp, i32 next}
//   root row      dense uni_lp[V], uni_next[V] (the unigram level)
//   per state     eos[S] = LM.Final and lm_ub[S] >= max_w log P(w | s) (pre-prune bound)
// State 0 is the root (empty context); it has no CSR arcs (the dense row replaces them).
// ---------------------------------------------------------------------------------------
// Device query structures derived from it:
//   rec[S][RW]    per-state record: {n_arc_levels, dense_row(-1 = none), cum_u, cum_root, ub, eos,
//                 sig (u64: bit lm_sig_bit(w) set for every token w with an arc at an arc level),
//                 then per arc level (context length >= 2): arc_off, arc_deg, cum}
//   dense[U][V]   rows of the length-1 contexts: {f32 value, next | found_at_level1 << 31}
struct LmHost {
    int32_t order = 0, V = 0, S = 0, start = 0;
    int32_t NL = 0, RW = 8, U = 0;
    std::vector<int32_t> st_hdr;   // 4 ints per state
    std::vector<uint16_t> arc_tok;
    std::vector<int32_t> arc_val;  // 2 ints per arc: f32 bits, next
    std::vector<float> uni_lp;
    std::vector<int32_t> uni_next;
    std::vector<float> eos, ub;
    std::vector<int32_t> rec;      // S * RW
    std::vector<int32_t> dense;    // U * V * 2
};

// 6-bit hash of a token for the record signature (Fibonacci hashing)
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int lm_sig_bit(int w) { return (int)(((uint32_t)w * 0x9E3779B1u) >> 26); }

struct LmDev {
    const int4* rec;               // S * RW/4 int4
    const int2* dense;
    const int4* arcs;              // {token, f32 logp bits, next state, 0}, sorted per state
    const float* uni_lp;
    const int32_t* uni_next;
    int32_t RW, V, start, NL;
    int64_t dense_bytes, arcs_bytes, rec_bytes;  // sizes (the L2 warm-up ranges)
};
constexpr int kMaxLmLevels = 6;    // arc levels (order - 2); order <= 8

// ---------------------------------------------------------------------------------------
// Boost device layout: full Aho-Corasick transition table [nodes x V] of {next, f32 delta}
// (delta = dC(v) + U(v) - U(u), reading R17), plus U[n] and maxd[n] = max_w delta(n, w).
// ---------------------------------------------------------------------------------------
struct BoostHost {
    int32_t V = 0, N = 0;
    std::vector<int32_t> tab;  // 2 ints per (node, token)
    std::vector<float> U, maxd;
    std::vector<uint64_t> sig;  // per node: lm_sig_bit(a) of every token a with δ(u, a) != δ(root, a)
};

struct BoostDev {
    const int2* tab;
    const float* U;
    const float* maxd;
    const unsigned long long* sig;  // exception signatures (BoostHost::sig)
    int32_t V;
    int64_t tab_bytes;
};

flexctc_status build_lm_host(const char* path, int32_t V, const char* const* syms, LmHost& out);
flexctc_status build_boost_host(const int32_t* toks, const int64_t* offs, int32_t n, float w, int32_t V,
                                BoostHost& out);

// host mirrors of the device queries (same arithmetic order), used by the inspection API
float lm_query_host(const LmHost& lm, int32_t s, int32_t w, int32_t* next);

// ---------------------------------------------------------------------------------------
// Decode kernel parameters
// ---------------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------------
// Frame records of the compaction pass (compact_kernel.cu, SURVEY §8(a) A1 "compact_frames"):
// 256 B per valid frame (b, t < L_b) at cmp + (b·T + t)·256:
//   f32 [0] D[blank], [1] floor, i32 [2] n, f32 [3] xthr, f64 at byte 16: lse (bf16-logits input; 0
//   for log-prob input), f32 val[32] at byte 32, u16 tok[32] at byte 160.
// tok[0..n) are the non-blank tokens listed for the frame, sorted by (D desc, token asc), with
// their D values; every non-blank token NOT listed has D <= floor (floor = +inf: no usable list,
// floor = -inf: every finite non-blank token is listed); a token is listed iff its raw input
// value (log-prob, or bf16 logit) is >= xthr.
// ---------------------------------------------------------------------------------------
constexpr int kCmpList = 32;
constexpr int kCmpBytes = 256;

constexpr int kChunk = 32;      // frames per backtrace chunk (chunk ancestors, §7.3 item 6)
constexpr int kMaxBeam = 256;   // parent index fits a u8
constexpr int kMaxVp1 = 8192;   // frame rows are staged in shared memory
constexpr int kStatsWords = 48; // u64 device counters at workspace + 64 B

struct DecodeParams {
    const float* log_probs;
    int64_t stride_b, stride_t;
    const int32_t* lengths;
    int32_t B, T, Vp1, K;
    float alpha_lm, alpha_bt, beta, theta;
    int32_t merge_mode, retract, fuse_rep;
    int32_t merge_first;  // reading R27: recombine before the TopK (merge_first_kernel.cu)
    int32_t use_lm, use_bt;
    int32_t solo_off;     // tuning/test switch: disable the beam-warp + helpers mode
    int32_t fast_off;     // A/B switch (FLEXCTC_FAST=0): disable the CTA kernel's settled-beam fast path
    // streamed input (flexctc_decode_host): frames [0, *ready) of every utterance have landed in
    // log_probs; the row loaders poll it (ld.acquire) before issuing a row. NULL = all resident.
    const uint32_t* ready;
    // wave > 0 (ragged host input): ready[0] counts the frames landed for the utterances at LPT
    // positions < wave (sent frame-major); ready[1] counts the utterances at positions wave, wave+1,
    // ... that have landed whole (sent in LPT order after the first wave)
    int32_t wave;
    // log_probs is a library-owned buffer with >= 16 B of slack on both sides of every row, so
    // rows are copied as whole 16-B blocks (no 4-B .ca copies that could cache stale sectors
    // while a chunk is still in flight)
    int32_t overread;
    LmDev lm;
    BoostDev bt;
    // workspace
    uint32_t* flags;      // [0] flags, [1] work queue
    unsigned long long* stats;  // [kStatsWords] device counters (flags + 64 B)
    int32_t* order;       // [B] utterances by length, longest first
    int32_t* len_c;       // [B] clamped lengths
    uint8_t* chunk_anc;   // [B][nch][K]
    uint8_t* bp_parent;   // [B][T][K]
    uint16_t* bp_label;   // [B][T][K]
    int32_t* align_ws;    // [B][T]
    float4* greedy_sum;   // [B][T] {d1, w1, d2, 0} frame summaries of the plain greedy path (K = 1)
    uint8_t* cmp;         // [B][T][kCmpBytes] frame records (K >= 2), NULL otherwise
    int32_t use_cmp;      // the records were written by the compaction pass of this decode (CTA kernel)
    int64_t* rowoff;      // [B + 1] prefix of the clamped lengths (compaction pass rows)
    const uint16_t* logits;  // bf16 logits input of the warp path (log_probs unused), or NULL
    int32_t nch;
    // outputs
    int32_t* out_tokens;
    int32_t* out_num;
    float* out_scores;
    int32_t* out_ts;
    int32_t* out_align;   // may alias align_ws
    int32_t nbest;        // 0 / 1: 1-best; N > 1: out_tokens [B][N][T], out_num / out_scores [B][N]
};

struct WorkspaceLayout {
    size_t flags, order, len_c, chunk_anc, bp_parent, bp_label, align_ws, greedy, cmp, rowoff, total;
    int32_t nch;
};
WorkspaceLayout workspace_layout(int32_t B, int32_t T, int32_t K);

// launches (beam_kernel.cu; K = 1 goes to launch_greedy in greedy_kernel.cu)
bool use_warp_path(const DecodeParams& p);  // K <= 32 warp path eligible (p.logits: bf16 input)
bool cta_logits_direct(const DecodeParams& p);  // bf16 logits read by the CTA kernel itself
// ev_start / ev_stop around the beam kernel, ev_cmp_start / ev_cmp_stop around the compaction pass
int launch_decode(const DecodeParams& p, void* stream, void* ev_start, void* ev_stop, std::string& err,
                  void* ev_cmp_start = nullptr, void* ev_cmp_stop = nullptr);
int launch_greedy(const DecodeParams& p, void* stream, void* ev_start, void* ev_stop, std::string& err);
// frame compaction pass (compact_kernel.cu): records of every valid row; rowoff by launch_rowoff
int launch_rowoff(const int32_t* len_c, int B, int64_t* rowoff, void* stream, std::string& err);
// exp(x) in fp64 for every bf16 bit pattern x (65536 entries, one per device, built on first use;
// NULL if it cannot be allocated): the log-sum-exp of bf16 rows by table loads (reading R25)
const double* bf16_exp_table(void* stream);
// byte ranges the decode's lookups hit at random (LM level-1 rows and arcs, boost table, ...),
// prefetched into L2 with evict-last priority
struct WarmRanges {
    const char* a[4] = {nullptr, nullptr, nullptr, nullptr};
    int64_t n[4] = {0, 0, 0, 0};
};
// warm (optional): the TMA pass interleaves the L2 warm-up of these ranges with its rows (no
// separate l2_warm launch); compact_fuses_warm tells whether the pass will take them
int launch_compact(const void* x, bool bf16, int64_t stride_b, int64_t stride_t, const int64_t* rowoff, int B, int T,
                   int Vp1, uint8_t* cmp, void* stream, std::string& err, const WarmRanges* warm = nullptr);
bool compact_fuses_warm(int Vp1, bool bf16);
// warp-per-utterance beam kernel (warp_beam_kernel.cu), K <= 32, after launch_compact
int launch_warp_beam(const DecodeParams& p, bool bf16, void* stream, void* ev_start, void* ev_stop, std::string& err);
size_t warp_beam_smem_per_warp(int Vp1, bool bf16, int nch);
// merge-before-TopK variant (merge_first_kernel.cu), after order_kernel
int launch_merge_first(const DecodeParams& p, void* stream, void* ev_start, void* ev_stop, std::string& err);
// input side (input_kernel.cu): log-softmax of bf16 logits into a dense fp32 [B][T][Vp1] buffer
// (frames [t0, t1) only; t1 = -1: every frame); preload_: force its module to load (see the .cu)
int preload_log_softmax_bf16();
// streamed host input: copy frames [t0, min(L_b, t1)) of every utterance from a device-mapped
// pinned host buffer to the device copy (same layout); preload_: load the module before the
// persistent kernel starts (a lazy module load would wait for it)
int preload_gather_rows();
int launch_gather_rows(const void* src_dev, void* dst, const int32_t* lengths, const int32_t* order, int n, int T,
                       int64_t row_bytes, int t0, int t1, int ctas, void* stream, std::string& err);
int launch_log_softmax_bf16(const uint16_t* x, int64_t stride_b, int64_t stride_t, const int32_t* lengths, int B,
                            int T, int Vp1, float* out, void* stream, std::string& err, int t0 = 0, int t1 = -1);

}  // namespace flexctc

struct flexctc_lm {
    int32_t device = -1;
    flexctc::LmHost host;
    void* dmem = nullptr;  // one device allocation holding every array
    size_t dbytes = 0;
    flexctc::LmDev dev{};
};

struct flexctc_boost {
    int32_t device = -1;
    flexctc::BoostHost host;
    void* dmem = nullptr;
    size_t dbytes = 0;
    flexctc::BoostDev dev{};
};
