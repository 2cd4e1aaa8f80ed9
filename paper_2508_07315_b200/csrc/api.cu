// C ABI of libflexctc (include/flexctc.h): validation, handle management, device upload,
// workspace layout, and the two launches of a decode. No compute happens on the host: the
// builders only lay out the LM / boost tables, and flexctc_decode refuses host memory.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "flexctc_internal.h"

namespace flexctc {

thread_local std::string g_error;
thread_local void* g_ev_start = nullptr;
thread_local void* g_ev_stop = nullptr;
thread_local void* g_ev_cmp_start = nullptr;  // stage 1: the frame compaction pass
thread_local void* g_ev_cmp_stop = nullptr;
thread_local const char* g_kernel = "";
void set_error(const std::string& msg) { g_error = msg; }
void set_kernel_name(const char* name) { g_kernel = name; }
flexctc_status fail(flexctc_status st, const std::string& msg) {
    g_error = msg;
    return st;
}

namespace {

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

flexctc_status cuda_fail(cudaError_t e, const char* what) {
    return fail(e == cudaErrorMemoryAllocation ? FLEXCTC_ERR_OOM : FLEXCTC_ERR_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

// one device allocation, arrays at 256-B aligned offsets
struct Upload {
    std::vector<std::pair<const void*, size_t>> parts;
    size_t add(const void* p, size_t n) {
        size_t off = 0;
        for (auto& q : parts) off += align256(q.second);
        parts.emplace_back(p, n);
        return off;
    }
    size_t total() const {
        size_t s = 0;
        for (auto& q : parts) s += align256(q.second);
        return s;
    }
};

flexctc_status upload(int device, Upload& up, void** dmem) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    const size_t tot = std::max<size_t>(up.total(), 256);
    e = cudaMalloc(dmem, tot);
    if (e != cudaSuccess) { cudaSetDevice(prev); return cuda_fail(e, "cudaMalloc"); }
    size_t off = 0;
    for (auto& q : up.parts) {
        if (q.second) {
            e = cudaMemcpy((char*)*dmem + off, q.first, q.second, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) { cudaFree(*dmem); *dmem = nullptr; cudaSetDevice(prev); return cuda_fail(e, "cudaMemcpy"); }
        }
        off += align256(q.second);
    }
    cudaSetDevice(prev);
    return FLEXCTC_OK;
}

bool is_device_ptr(const void* p, int dev) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    if (a.type == cudaMemoryTypeManaged) return true;
    return a.type == cudaMemoryTypeDevice && a.device == dev;
}

}  // namespace

WorkspaceLayout workspace_layout(int32_t B, int32_t T, int32_t K) {
    WorkspaceLayout w{};
    w.nch = (T + kChunk - 1) / kChunk;
    if (w.nch < 1) w.nch = 1;
    size_t o = 0;
    w.flags = o; o += align256(64 + 8 * kStatsWords);
    w.order = o; o += align256(4 * (size_t)B);
    w.len_c = o; o += align256(4 * (size_t)B);
    w.chunk_anc = o; o += align256((size_t)B * w.nch * K);
    w.bp_parent = o; o += align256((size_t)B * T * K);
    w.bp_label = o; o += align256((size_t)B * T * K * 2);
    w.align_ws = o; o += align256((size_t)B * T * 4);
    w.greedy = o; o += K == 1 ? align256((size_t)B * T * 16) : 0;  // plain greedy frame summaries
    const bool warp = K >= 2;  // frame records + row prefix (compaction pass; every beam path K >= 2)
    w.cmp = o; o += warp ? align256((size_t)B * T * kCmpBytes) : 0;
    w.rowoff = o; o += warp ? align256(8 * ((size_t)B + 1)) : 0;
    w.total = o;
    return w;
}

}  // namespace flexctc

using namespace flexctc;

extern "C" {

const char* flexctc_last_error(void) { return g_error.c_str(); }
const char* flexctc_version(void) { return "flexctc-b200 0.2 (sm_100a)"; }
const char* flexctc_last_kernel(void) { return g_kernel; }

flexctc_status flexctc_lm_load(const char* arpa_path, int32_t vocab_size, const char* const* token_symbols,
                               int32_t device, flexctc_lm** out) {
    if (!out) return fail(FLEXCTC_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!arpa_path) return fail(FLEXCTC_ERR_INVALID_ARG, "arpa_path is NULL");
    auto* lm = new flexctc_lm();
    flexctc_status st = build_lm_host(arpa_path, vocab_size, token_symbols, lm->host);
    if (st != FLEXCTC_OK) { delete lm; return st; }
    lm->device = device;
    if (device >= 0) {
        const LmHost& h = lm->host;
        Upload up;
        if (h.NL > kMaxLmLevels) { delete lm; return fail(FLEXCTC_ERR_CAPACITY, "LM order > 8"); }
        size_t o_rec = up.add(h.rec.data(), h.rec.size() * 4);
        size_t o_den = up.add(h.dense.data(), h.dense.size() * 4);
        std::vector<int32_t> arcs4(h.arc_tok.size() * 4, 0);
        for (size_t k = 0; k < h.arc_tok.size(); ++k) {
            arcs4[4 * k] = h.arc_tok[k];
            arcs4[4 * k + 1] = h.arc_val[2 * k];
            arcs4[4 * k + 2] = h.arc_val[2 * k + 1];
        }
        size_t o_arc = up.add(arcs4.data(), arcs4.size() * 4);
        size_t o_ulp = up.add(h.uni_lp.data(), h.uni_lp.size() * 4);
        size_t o_unx = up.add(h.uni_next.data(), h.uni_next.size() * 4);
        st = upload(device, up, &lm->dmem);
        if (st != FLEXCTC_OK) { delete lm; return st; }
        lm->dbytes = up.total();
        char* d = (char*)lm->dmem;
        lm->dev.rec = (const int4*)(d + o_rec);
        lm->dev.dense = (const int2*)(d + o_den);
        lm->dev.arcs = (const int4*)(d + o_arc);
        lm->dev.dense_bytes = (int64_t)h.dense.size() * 4;
        lm->dev.arcs_bytes = (int64_t)arcs4.size() * 4;
        lm->dev.rec_bytes = (int64_t)h.rec.size() * 4;
        lm->dev.uni_lp = (const float*)(d + o_ulp);
        lm->dev.uni_next = (const int32_t*)(d + o_unx);
        lm->dev.RW = h.RW;
        lm->dev.V = h.V;
        lm->dev.NL = h.NL;
        lm->dev.start = h.start;
    }
    *out = lm;
    return FLEXCTC_OK;
}

void flexctc_lm_free(flexctc_lm* lm) {
    if (!lm) return;
    if (lm->dmem) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(lm->device);
        cudaFree(lm->dmem);
        cudaSetDevice(prev);
    }
    delete lm;
}

flexctc_status flexctc_lm_get_info(const flexctc_lm* lm, flexctc_lm_info* info) {
    if (!lm || !info) return fail(FLEXCTC_ERR_INVALID_ARG, "NULL argument");
    info->order = lm->host.order;
    info->vocab_size = lm->host.V;
    info->n_states = lm->host.S;
    info->start_state = lm->host.start;
    info->n_arcs = (int64_t)lm->host.arc_tok.size();
    info->device_bytes = (int64_t)lm->dbytes;
    return FLEXCTC_OK;
}

flexctc_status flexctc_lm_host_query(const flexctc_lm* lm, int32_t state, int32_t token, float* logp,
                                     int32_t* next_state) {
    if (!lm || !logp || !next_state) return fail(FLEXCTC_ERR_INVALID_ARG, "NULL argument");
    if (state < 0 || state >= lm->host.S) return fail(FLEXCTC_ERR_INVALID_ARG, "state out of range");
    if (token == -1) {
        *logp = lm->host.eos[state];
        *next_state = state;
        return FLEXCTC_OK;
    }
    if (token < 0 || token >= lm->host.V) return fail(FLEXCTC_ERR_INVALID_ARG, "token out of range");
    *logp = lm_query_host(lm->host, state, token, next_state);
    return FLEXCTC_OK;
}

flexctc_status flexctc_lm_host_query_batch(const flexctc_lm* lm, int64_t n, const int32_t* states,
                                           const int32_t* tokens, float* logp, int32_t* next_state) {
    if (!lm || n < 0 || (n > 0 && (!states || !tokens || !logp || !next_state)))
        return fail(FLEXCTC_ERR_INVALID_ARG, "NULL argument");
    for (int64_t i = 0; i < n; ++i) {
        const flexctc_status st = flexctc_lm_host_query(lm, states[i], tokens[i], &logp[i], &next_state[i]);
        if (st != FLEXCTC_OK) return st;
    }
    return FLEXCTC_OK;
}

flexctc_status flexctc_lm_host_bound(const flexctc_lm* lm, int32_t state, float* ub, float* eos) {
    if (!lm || !ub || !eos) return fail(FLEXCTC_ERR_INVALID_ARG, "NULL argument");
    if (state < 0 || state >= lm->host.S) return fail(FLEXCTC_ERR_INVALID_ARG, "state out of range");
    *ub = lm->host.ub[state];
    *eos = lm->host.eos[state];
    return FLEXCTC_OK;
}

flexctc_status flexctc_boost_build(const int32_t* tokens, const int64_t* offsets, int32_t n_phrases,
                                   float token_weight, int32_t vocab_size, int32_t device, flexctc_boost** out) {
    if (!out) return fail(FLEXCTC_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    auto* bt = new flexctc_boost();
    flexctc_status st = build_boost_host(tokens, offsets, n_phrases, token_weight, vocab_size, bt->host);
    if (st != FLEXCTC_OK) { delete bt; return st; }
    bt->device = device;
    if (device >= 0) {
        const BoostHost& h = bt->host;
        Upload up;
        size_t o_tab = up.add(h.tab.data(), h.tab.size() * 4);
        size_t o_u = up.add(h.U.data(), h.U.size() * 4);
        size_t o_m = up.add(h.maxd.data(), h.maxd.size() * 4);
        size_t o_s = up.add(h.sig.data(), h.sig.size() * 8);
        st = upload(device, up, &bt->dmem);
        if (st != FLEXCTC_OK) { delete bt; return st; }
        bt->dbytes = up.total();
        char* d = (char*)bt->dmem;
        bt->dev.tab = (const int2*)(d + o_tab);
        bt->dev.tab_bytes = (int64_t)h.tab.size() * 4;
        bt->dev.U = (const float*)(d + o_u);
        bt->dev.maxd = (const float*)(d + o_m);
        bt->dev.sig = (const unsigned long long*)(d + o_s);
        bt->dev.V = h.V;
    }
    *out = bt;
    return FLEXCTC_OK;
}

void flexctc_boost_free(flexctc_boost* bt) {
    if (!bt) return;
    if (bt->dmem) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(bt->device);
        cudaFree(bt->dmem);
        cudaSetDevice(prev);
    }
    delete bt;
}

flexctc_status flexctc_boost_host_query(const flexctc_boost* bt, int32_t node, int32_t token, float* delta,
                                        int32_t* next_node, float* U_node) {
    if (!bt || !delta || !next_node || !U_node) return fail(FLEXCTC_ERR_INVALID_ARG, "NULL argument");
    const BoostHost& h = bt->host;
    if (node < 0 || node >= h.N || token < 0 || token >= h.V) return fail(FLEXCTC_ERR_INVALID_ARG, "node/token out of range");
    const size_t e = ((size_t)node * h.V + token) * 2;
    *next_node = h.tab[e];
    memcpy(delta, &h.tab[e + 1], 4);
    *U_node = h.U[node];
    return FLEXCTC_OK;
}

flexctc_status flexctc_boost_host_query_batch(const flexctc_boost* bt, int64_t n, const int32_t* nodes,
                                              const int32_t* tokens, float* delta, int32_t* next_node) {
    if (!bt || n < 0 || (n > 0 && (!nodes || !tokens || !delta || !next_node)))
        return fail(FLEXCTC_ERR_INVALID_ARG, "NULL argument");
    float U = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
        const flexctc_status st = flexctc_boost_host_query(bt, nodes[i], tokens[i], &delta[i], &next_node[i], &U);
        if (st != FLEXCTC_OK) return st;
    }
    return FLEXCTC_OK;
}

flexctc_status flexctc_boost_host_signature(const flexctc_boost* bt, int32_t node, uint64_t* sig) {
    if (!bt || !sig) return fail(FLEXCTC_ERR_INVALID_ARG, "NULL argument");
    if (node < 0 || node >= bt->host.N) return fail(FLEXCTC_ERR_INVALID_ARG, "node out of range");
    *sig = bt->host.sig[node];
    return FLEXCTC_OK;
}

flexctc_status flexctc_boost_num_nodes(const flexctc_boost* bt, int32_t* n_nodes) {
    if (!bt || !n_nodes) return fail(FLEXCTC_ERR_INVALID_ARG, "NULL argument");
    *n_nodes = bt->host.N;
    return FLEXCTC_OK;
}

size_t flexctc_workspace_bytes(int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg) {
    (void)Vp1;
    if (!cfg || B < 0 || T < 0 || cfg->beam < 1) return 0;
    return workspace_layout(B, T, cfg->beam).total;
}

size_t flexctc_logits_workspace_bytes(int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg) {
    if (!cfg || B < 0 || T < 0 || Vp1 < 2 || cfg->beam < 1) return 0;
    return workspace_layout(B, T, cfg->beam).total + (((size_t)B * T * Vp1 * 4 + 255) & ~size_t(255));
}

static flexctc_status validate_cfg(const flexctc_config* cfg) {
    if (!cfg) return fail(FLEXCTC_ERR_INVALID_ARG, "cfg is NULL");
    if (cfg->beam < 1) return fail(FLEXCTC_ERR_INVALID_ARG, "beam must be >= 1");
    if (cfg->beam > kMaxBeam) return fail(FLEXCTC_ERR_CAPACITY, "beam > 256");
    if (!(cfg->theta >= 0.0f)) return fail(FLEXCTC_ERR_INVALID_ARG, "theta must be >= 0 (or +inf)");
    if (cfg->merge_mode != 0 && cfg->merge_mode != 1) return fail(FLEXCTC_ERR_INVALID_ARG, "merge_mode must be 0 or 1");
    if (cfg->fuse_repeats != 0 && cfg->fuse_repeats != 1) return fail(FLEXCTC_ERR_INVALID_ARG, "fuse_repeats must be 0 or 1");
    if (cfg->merge_first != 0 && cfg->merge_first != 1) return fail(FLEXCTC_ERR_INVALID_ARG, "merge_first must be 0 or 1");
    if (!std::isfinite(cfg->alpha_lm) || !std::isfinite(cfg->alpha_bt) || !std::isfinite(cfg->beta))
        return fail(FLEXCTC_ERR_INVALID_ARG, "alpha/beta must be finite");
    return FLEXCTC_OK;
}

// flexctc_decode plus the streamed-input fields of DecodeParams (ready, overread), which only
// flexctc_decode_host sets.
static flexctc_status decode_impl(const float* log_probs, int64_t stride_b, int64_t stride_t, const int32_t* lengths,
                                  int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg, const flexctc_lm* lm,
                                  const flexctc_boost* boost, void* workspace, size_t workspace_bytes,
                                  flexctc_stream stream, int32_t* out_tokens, int32_t* out_num_tokens,
                                  float* out_scores, int32_t* out_timestamps, int32_t* out_alignment,
                                  const uint32_t* ready, int overread, int32_t nbest = 1,
                                  const uint16_t* logits = nullptr, int32_t wave = 0) {
    flexctc_status st = validate_cfg(cfg);
    if (st != FLEXCTC_OK) return st;
    if (nbest < 1 || nbest > cfg->beam) return fail(FLEXCTC_ERR_INVALID_ARG, "nbest must be in [1, beam]");
    if (cfg->merge_first && (nbest > 1 || logits)) return fail(FLEXCTC_ERR_INVALID_ARG, "merge_first: 1-best over log-probs only");
    if (B < 0 || T < 0) return fail(FLEXCTC_ERR_INVALID_ARG, "B and T must be >= 0");
    if (Vp1 < 2) return fail(FLEXCTC_ERR_INVALID_ARG, "Vp1 must be >= 2");
    if (Vp1 > kMaxVp1) return fail(FLEXCTC_ERR_CAPACITY, "Vp1 > 8192");
    // the stride of a size-1 axis is never used (torch / numpy give such axes arbitrary strides)
    if ((T > 1 && stride_t < Vp1) || (B > 1 && stride_b < (int64_t)std::max(T, 1) * (T > 1 ? stride_t : (int64_t)Vp1)) ||
        stride_t < 0 || stride_b < 0)
        return fail(FLEXCTC_ERR_INVALID_ARG, "strides overlap rows");
    if ((int64_t)Vp1 * cfg->beam >= (int64_t)0xffffffff) return fail(FLEXCTC_ERR_CAPACITY, "K*Vp1 too large");
    const WorkspaceLayout wl = workspace_layout(B, T, cfg->beam);
    const size_t need = wl.total + (logits ? ((size_t)B * T * Vp1 * 4 + 255) & ~size_t(255) : 0);
    if (!workspace || workspace_bytes < need)
        return fail(FLEXCTC_ERR_CAPACITY, logits ? "workspace smaller than flexctc_logits_workspace_bytes()"
                                                 : "workspace smaller than flexctc_workspace_bytes()");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (B == 0) return FLEXCTC_OK;
    // T = 0: the [B, T] arrays are empty and may be NULL (nothing is read or written there)
    auto dev_bt = [&](const void* q, bool required) { return T == 0 ? true : (q ? is_device_ptr(q, dev) : !required); };
    if (!dev_bt(logits ? (const void*)logits : (const void*)log_probs, true) || !is_device_ptr(lengths, dev) || !is_device_ptr(workspace, dev) ||
        !dev_bt(out_tokens, true) || !is_device_ptr(out_num_tokens, dev) || !is_device_ptr(out_scores, dev) ||
        !dev_bt(out_timestamps, false) || !dev_bt(out_alignment, false))
        return fail(FLEXCTC_ERR_INVALID_ARG, "every buffer must be device memory of the current device (no CPU path)");
    if (lm) {
        if (lm->device != dev || !lm->dmem) return fail(FLEXCTC_ERR_INVALID_ARG, "LM handle belongs to another device");
        if (lm->host.V != Vp1 - 1) return fail(FLEXCTC_ERR_INVALID_ARG, "LM vocab_size != Vp1-1");
    }
    if (boost) {
        if (boost->device != dev || !boost->dmem) return fail(FLEXCTC_ERR_INVALID_ARG, "boost handle belongs to another device");
        if (boost->host.V != Vp1 - 1) return fail(FLEXCTC_ERR_INVALID_ARG, "boost vocab_size != Vp1-1");
    }
    DecodeParams p{};
    p.log_probs = log_probs;
    p.stride_b = stride_b;
    p.stride_t = stride_t;
    p.lengths = lengths;
    p.B = B; p.T = T; p.Vp1 = Vp1; p.K = cfg->beam;
    p.alpha_lm = cfg->alpha_lm; p.alpha_bt = cfg->alpha_bt; p.beta = cfg->beta; p.theta = cfg->theta;
    p.merge_mode = cfg->merge_mode; p.retract = cfg->retract_boost_at_eos; p.fuse_rep = cfg->fuse_repeats ? 1 : 0;
    p.merge_first = cfg->merge_first ? 1 : 0;
    p.use_lm = lm != nullptr; p.use_bt = boost != nullptr;
    if (lm) p.lm = lm->dev;
    if (boost) p.bt = boost->dev;
    char* w = (char*)workspace;
    p.flags = (uint32_t*)(w + wl.flags);
    p.stats = (unsigned long long*)(w + wl.flags + 64);
    p.order = (int32_t*)(w + wl.order);
    p.len_c = (int32_t*)(w + wl.len_c);
    p.chunk_anc = (uint8_t*)(w + wl.chunk_anc);
    p.bp_parent = (uint8_t*)(w + wl.bp_parent);
    p.bp_label = (uint16_t*)(w + wl.bp_label);
    p.align_ws = (int32_t*)(w + wl.align_ws);
    p.greedy_sum = cfg->beam == 1 ? (float4*)(w + wl.greedy) : nullptr;
    const bool warp_ws = cfg->beam >= 2;
    p.cmp = warp_ws ? (uint8_t*)(w + wl.cmp) : nullptr;
    p.rowoff = warp_ws ? (int64_t*)(w + wl.rowoff) : nullptr;
    p.nch = wl.nch;
    p.out_tokens = out_tokens; p.out_num = out_num_tokens; p.out_scores = out_scores;
    p.out_ts = out_timestamps; p.out_align = out_alignment;
    p.ready = ready;
    p.wave = ready ? wave : 0;
    p.overread = overread;
    p.nbest = nbest;
    std::string err;
    p.logits = logits;
    if (logits && !use_warp_path(p) && !cta_logits_direct(p)) {
        // bf16 logits, K = 1 or K > 32: a bandwidth-bound log-softmax pass (R25) into the
        // workspace's dense fp32 [B][T][Vp1] region, then the decode of those log-probs (the
        // K <= 32 warp path instead fuses the log-softmax into its compaction pass)
        p.logits = nullptr;
        float* Dw = (float*)((char*)workspace + wl.total);
        const int rc0 = launch_log_softmax_bf16(logits, stride_b, stride_t, lengths, B, T, Vp1, Dw, (void*)stream, err);
        if (rc0 == 2) return fail(FLEXCTC_ERR_CAPACITY, err);
        if (rc0 != 0) return fail(FLEXCTC_ERR_CUDA, err);
        p.log_probs = Dw;
        p.stride_b = (int64_t)T * Vp1;
        p.stride_t = Vp1;
    }
    int rc = launch_decode(p, (void*)stream, g_ev_start, g_ev_stop, err, g_ev_cmp_start, g_ev_cmp_stop);
    if (rc == 2) return fail(FLEXCTC_ERR_CAPACITY, err);
    if (rc != 0) return fail(FLEXCTC_ERR_CUDA, err);
    return FLEXCTC_OK;
}

flexctc_status flexctc_decode(const float* log_probs, int64_t stride_b, int64_t stride_t, const int32_t* lengths,
                              int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg, const flexctc_lm* lm,
                              const flexctc_boost* boost, void* workspace, size_t workspace_bytes,
                              flexctc_stream stream, int32_t* out_tokens, int32_t* out_num_tokens,
                              float* out_scores, int32_t* out_timestamps, int32_t* out_alignment) {
    return decode_impl(log_probs, stride_b, stride_t, lengths, B, T, Vp1, cfg, lm, boost, workspace, workspace_bytes,
                       stream, out_tokens, out_num_tokens, out_scores, out_timestamps, out_alignment, nullptr, 0);
}

flexctc_status flexctc_decode_nbest(const float* log_probs, int64_t stride_b, int64_t stride_t,
                                    const int32_t* lengths, int32_t B, int32_t T, int32_t Vp1,
                                    const flexctc_config* cfg, const flexctc_lm* lm, const flexctc_boost* boost,
                                    void* workspace, size_t workspace_bytes, flexctc_stream stream, int32_t nbest,
                                    int32_t* out_tokens, int32_t* out_num_tokens, float* out_scores,
                                    int32_t* out_timestamps) {
    return decode_impl(log_probs, stride_b, stride_t, lengths, B, T, Vp1, cfg, lm, boost, workspace, workspace_bytes,
                       stream, out_tokens, out_num_tokens, out_scores, out_timestamps, nullptr, nullptr, 0, nbest);
}

flexctc_status flexctc_decode_logits_bf16(const uint16_t* logits, int64_t stride_b, int64_t stride_t,
                                          const int32_t* lengths, int32_t B, int32_t T, int32_t Vp1,
                                          const flexctc_config* cfg, const flexctc_lm* lm,
                                          const flexctc_boost* boost, void* workspace, size_t workspace_bytes,
                                          flexctc_stream stream, int32_t* out_tokens, int32_t* out_num_tokens,
                                          float* out_scores, int32_t* out_timestamps, int32_t* out_alignment) {
    if (T > 0 && !logits) return fail(FLEXCTC_ERR_INVALID_ARG, "logits is NULL");
    return decode_impl(nullptr, stride_b, stride_t, lengths, B, T, Vp1, cfg, lm, boost, workspace, workspace_bytes,
                       stream, out_tokens, out_num_tokens, out_scores, out_timestamps, out_alignment, nullptr, 0, 1,
                       logits);
}

void flexctc_set_profile_events(void* ev_start, void* ev_stop) {
    g_ev_start = ev_start;
    g_ev_stop = ev_stop;
}

flexctc_status flexctc_set_stage_events(int32_t stage, void* ev_start, void* ev_stop) {
    if (stage == 0) {
        g_ev_start = ev_start;
        g_ev_stop = ev_stop;
    } else if (stage == 1) {
        g_ev_cmp_start = ev_start;
        g_ev_cmp_stop = ev_stop;
    } else {
        return fail(FLEXCTC_ERR_INVALID_ARG, "unknown stage");
    }
    return FLEXCTC_OK;
}

flexctc_status flexctc_get_stats(const void* workspace, uint64_t* out, int32_t n) {
    if (!workspace || !out || n < 0) return fail(FLEXCTC_ERR_INVALID_ARG, "bad argument");
    const int k = n < kStatsWords ? n : kStatsWords;
    cudaError_t e = cudaMemcpy(out, (const char*)workspace + 64, 8 * (size_t)k, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy");
    return FLEXCTC_OK;
}

flexctc_status flexctc_check(const void* workspace, uint32_t* device_flags) {
    if (!workspace || !device_flags) return fail(FLEXCTC_ERR_INVALID_ARG, "NULL argument");
    cudaError_t e = cudaMemcpy(device_flags, workspace, sizeof(uint32_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy");
    return FLEXCTC_OK;
}

size_t flexctc_host_scratch_bytes(int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg) {
    if (!cfg || B < 0 || T < 0 || Vp1 < 2 || cfg->beam < 1) return 0;
    size_t s = align256((size_t)B * T * Vp1 * 4 + 16) + align256((size_t)B * 4) * 2 + 256;  // D, lengths, LPT order
    s += align256((size_t)B * T * 4) * 2 + align256((size_t)B * 4) * 2;
    s += workspace_layout(B, T, cfg->beam).total;
    return s;
}

size_t flexctc_host_scratch_bytes_bf16(int32_t B, int32_t T, int32_t Vp1, const flexctc_config* cfg) {
    const size_t s = flexctc_host_scratch_bytes(B, T, Vp1, cfg);
    return s ? s + align256((size_t)B * T * Vp1 * 2 + 16) : 0;  // + the bf16 logits copy
}

}  // extern "C"

namespace flexctc {
namespace {

// Per-thread resources of the streamed host path: a non-blocking copy stream, two events, and
// cuStreamWriteValue32 (a stream memory operation: the front end writes the "frames ready"
// word after each chunk's copy without occupying an SM, so it cannot be starved by the
// persistent kernel). Resolved through the runtime, no link against libcuda.
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct HostPath {
    int device = -1;
    cudaStream_t copy = nullptr;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    WriteValue32Fn write32 = nullptr;
    bool memops = false;
};
thread_local HostPath g_host;

bool host_path_init(int dev) {
    if (g_host.device == dev) return g_host.memops;
    g_host = HostPath{};
    g_host.device = dev;
    if (cudaStreamCreateWithFlags(&g_host.copy, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&g_host.ev_a, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g_host.ev_b, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn) {
        g_host.write32 = (WriteValue32Fn)fn;
        g_host.memops = true;  // 32-bit stream memory operations are always supported (CUDA >= 12)
    }
    cudaGetLastError();
    return g_host.memops;
}

// Frame chunks of the streamed copy: small first chunks so the decode starts early, then 32.
std::vector<int> chunk_ends(int T) {
    std::vector<int> e;
    int t = 0, c = 4;
    while (t < T) {
        t = std::min(T, t + c);
        e.push_back(t);
        c = std::min(32, 2 * c);
    }
    return e;
}

}  // namespace
}  // namespace flexctc

extern "C" {

int32_t flexctc_host_streaming(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return 0; }
    return host_path_init(dev) && !getenv("FLEXCTC_NO_STREAM_INPUT") ? 1 : 0;
}

}  // extern "C"

namespace flexctc {
namespace {

// flexctc_decode_host / flexctc_decode_host_bf16: H2D (streamed in frame chunks for K > 1, so the
// copy overlaps the frame recurrence), decode, D2H, sync. bf16 logits are normalised on the
// device (reading R25) into the fp32 log-prob buffer, chunk by chunk on the copy stream before
// each chunk's "frames ready" signal; the PCIe transfer is 2 B per logit.
flexctc_status decode_host_impl(const void* x_host, bool bf16, const int32_t* lengths_host, int32_t B, int32_t T,
                                int32_t Vp1, const flexctc_config* cfg, const flexctc_lm* lm,
                                const flexctc_boost* boost, void* device_scratch, size_t scratch_bytes,
                                flexctc_stream stream, int32_t* out_tokens, int32_t* out_num_tokens,
                                float* out_scores, int32_t* out_timestamps, uint32_t* out_flags) {
    if (out_flags) *out_flags = 0;
    flexctc_status st = validate_cfg(cfg);
    if (st != FLEXCTC_OK) return st;
    if (B < 0 || T < 0 || Vp1 < 2) return fail(FLEXCTC_ERR_INVALID_ARG, "bad shape");
    const size_t need = bf16 ? flexctc_host_scratch_bytes_bf16(B, T, Vp1, cfg) : flexctc_host_scratch_bytes(B, T, Vp1, cfg);
    if (!device_scratch || scratch_bytes < need) return fail(FLEXCTC_ERR_CAPACITY, "device_scratch too small");
    if (!x_host || !lengths_host || !out_tokens || !out_num_tokens || !out_scores)
        return fail(FLEXCTC_ERR_INVALID_ARG, "NULL argument");
    if (B == 0) return FLEXCTC_OK;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t s = (cudaStream_t)stream;
    char* d = (char*)(((uintptr_t)device_scratch + 255) & ~(uintptr_t)255);
    size_t o = 0;
    float* dD = (float*)(d + o); o += align256((size_t)B * T * Vp1 * 4 + 16);  // + 16 B slack (overread)
    int32_t* dL = (int32_t*)(d + o); o += align256((size_t)B * 4);
    int32_t* dOrd = (int32_t*)(d + o); o += align256((size_t)B * 4);  // LPT order (ragged streamed input)
    int32_t* dTok = (int32_t*)(d + o); o += align256((size_t)B * T * 4);
    int32_t* dTs = (int32_t*)(d + o); o += align256((size_t)B * T * 4);
    int32_t* dN = (int32_t*)(d + o); o += align256((size_t)B * 4);
    float* dS = (float*)(d + o); o += align256((size_t)B * 4);
    uint16_t* dX = nullptr;  // bf16 logits copy
    if (bf16) { dX = (uint16_t*)(d + o); o += align256((size_t)B * T * Vp1 * 2 + 16); }
    void* ws = d + o;
    const size_t wsb = scratch_bytes - (size_t)(d - (char*)device_scratch) - o;
    const WorkspaceLayout wl = workspace_layout(B, T, cfg->beam);
    const size_t esz = bf16 ? 2 : 4;
    char* dIn = bf16 ? (char*)dX : (char*)dD;
    // Streamed input: the persistent beam kernel starts at once and each row loader waits for
    // its frame chunk (a "frames ready" word in the workspace, written by the copy stream after
    // every chunk), so the host->device copy overlaps the frame recurrence. Only frames
    // t < lengths[b] are copied (the padding is never read). K = 1 and configurations without
    // stream memory operations copy everything first; so does bf16 input unless the batch leaves
    // SMs free for the per-chunk normalisation next to the persistent kernel (B < #SMs).
    const bool streamed = host_path_init(dev) && cfg->beam > 1 && T > 0 && (!bf16 || B < nsm) &&
                          !getenv("FLEXCTC_NO_STREAM_INPUT");  // test switch: copy everything, then decode
    e = cudaMemcpyAsync(dL, lengths_host, (size_t)B * 4, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync H2D");
    uint32_t* ready = nullptr;
    std::string err;
    if (streamed && bf16 && preload_log_softmax_bf16())
        return fail(FLEXCTC_ERR_CUDA, "cannot load the bf16 normalisation kernel");
    // Ragged batches: frames of the utterances still live in a chunk are gathered by a small kernel
    // that reads the caller's buffer over PCIe when it is pinned (device-mapped); one 2D copy per
    // run of live utterances otherwise (many copy calls for LibriSpeech-shaped lengths)
    const char* x_dev = nullptr;
    if (streamed) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, x_host) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer &&
            ((uintptr_t)pa.devicePointer & 15) == 0)  // same 16-B alignment as the device copy
            x_dev = (const char*)pa.devicePointer;
        cudaGetLastError();
        if (x_dev && preload_gather_rows()) x_dev = nullptr;
    }
    // Ragged fp32 input from a device-mapped buffer: the first wave of utterances (LPT positions
    // < #SMs, the ones the persistent kernel starts with) is sent frame-major, the rest whole in
    // LPT order, exactly when the kernel's work queue reaches them (a frame-major stream over all
    // utterances would feed utterances that start much later and starve the first wave).
    int Lmin = T;
    for (int b = 0; b < B; ++b) Lmin = std::min(Lmin, std::min(std::max(lengths_host[b], 0), T));
    int wave = 0;
    std::vector<int32_t> ord;
    if (streamed && x_dev && !bf16 && Lmin < T && B > nsm) {
        wave = nsm;
        ord.resize(B);
        for (int b = 0; b < B; ++b) ord[b] = b;
        if (B <= 16384)  // order_kernel's rule: length desc, ties to the lower index (identity above)
            std::stable_sort(ord.begin(), ord.end(), [&](int a, int c) {
                return std::min(std::max(lengths_host[a], 0), T) > std::min(std::max(lengths_host[c], 0), T);
            });
        e = cudaMemcpyAsync(dOrd, ord.data(), (size_t)B * 4, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync H2D");
    }
    if (streamed) {
        ready = (uint32_t*)((char*)ws + wl.flags + 64 + 8 * kStatsWords);
        e = cudaMemsetAsync(ready, 0, 8, s);
        if (e == cudaSuccess) e = cudaEventRecord(g_host.ev_a, s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(g_host.copy, g_host.ev_a, 0);
        if (e != cudaSuccess) return cuda_fail(e, "stream setup");
    } else {
        e = cudaMemcpyAsync(dIn, x_host, (size_t)B * T * Vp1 * esz, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync H2D");
        if (bf16) {
            const int rc = launch_log_softmax_bf16(dX, (int64_t)T * Vp1, Vp1, dL, B, T, Vp1, dD, (void*)s, err);
            if (rc) return fail(rc == 2 ? FLEXCTC_ERR_CAPACITY : FLEXCTC_ERR_CUDA, err);
        }
    }
    st = decode_impl(dD, (int64_t)T * Vp1, Vp1, dL, B, T, Vp1, cfg, lm, boost, ws, wsb, stream, dTok, dN, dS,
                     out_timestamps ? dTs : nullptr, nullptr, ready, 1, 1, nullptr, wave);
    // (the pageable `ord` upload above returned once staged: the vector may go)
    if (st != FLEXCTC_OK) {
        if (streamed) cudaStreamSynchronize(s);
        return st;
    }
    if (streamed) {
        // chunk c: frames [t0, t1) of every utterance with L_b > t0 (rows of one utterance are
        // contiguous), [bf16: normalised into dD], then ready = t1
        const size_t row = (size_t)Vp1 * esz;
        const char* xh = (const char*)x_host;
        int t0 = 0;
        int Tw = T;  // frames of the first wave
        if (wave) {
            Tw = 0;
            for (int u = 0; u < wave; ++u) Tw = std::max(Tw, std::min(std::max(lengths_host[ord[u]], 0), T));
        }
        for (int t1 : chunk_ends(Tw)) {
            if (t1 <= Lmin && !wave) {  // every utterance needs the whole chunk: one 2D copy
                e = cudaMemcpy2DAsync(dIn + (size_t)t0 * row, (size_t)T * row, xh + (size_t)t0 * row,
                                      (size_t)T * row, row * (size_t)(t1 - t0), (size_t)B, cudaMemcpyHostToDevice,
                                      g_host.copy);
            } else if (x_dev) {
                // ragged, pinned: one gather launch copies the chunk's valid frames of every
                // utterance (of the first wave when waved)
                if (launch_gather_rows(x_dev, dIn, dL, wave ? dOrd : nullptr, wave ? wave : B, T, (int64_t)row, t0, t1,
                                       32, (void*)g_host.copy, err))
                    e = cudaErrorUnknown;
            } else {
                // ragged: one 2D copy of the whole chunk per maximal run of consecutive utterances
                // with L_b > t0 (an utterance ending inside the chunk also gets its padding rows
                // [L_b, t1) of the caller's buffer: never read by the decode)
                for (int b = 0; b < B && e == cudaSuccess;) {
                    auto alive = [&](int i) { return std::min(std::max(lengths_host[i], 0), T) > t0; };
                    if (!alive(b)) { ++b; continue; }
                    int b1 = b + 1;
                    while (b1 < B && alive(b1)) ++b1;
                    const size_t off = ((size_t)b * T + t0) * row;
                    e = cudaMemcpy2DAsync(dIn + off, (size_t)T * row, xh + off, (size_t)T * row,
                                          row * (size_t)(t1 - t0), (size_t)(b1 - b), cudaMemcpyHostToDevice, g_host.copy);
                    b = b1;
                }
            }
            if (e == cudaSuccess && bf16 &&
                launch_log_softmax_bf16(dX, (int64_t)T * Vp1, Vp1, dL, B, T, Vp1, dD, (void*)g_host.copy, err, t0, t1))
                e = cudaErrorUnknown;
            if (e == cudaSuccess &&
                g_host.write32((CUstream)g_host.copy, (CUdeviceptr)ready, (cuuint32_t)t1, 0) != CUDA_SUCCESS)
                e = cudaErrorUnknown;
            if (e != cudaSuccess) break;
            t0 = t1;
        }
        // the later utterances whole, in LPT order, in growing groups; ready[1] = how many landed
        for (int u0 = wave, g = 4; wave && u0 < B && e == cudaSuccess; u0 += g, g = std::min(64, 2 * g)) {
            const int u1 = std::min(B, u0 + g);
            if (launch_gather_rows(x_dev, dIn, dL, dOrd + u0, u1 - u0, T, (int64_t)row, 0, T, 32, (void*)g_host.copy, err))
                e = cudaErrorUnknown;
            if (e == cudaSuccess && g_host.write32((CUstream)g_host.copy, (CUdeviceptr)(ready + 1),
                                                   (cuuint32_t)(u1 - wave), 0) != CUDA_SUCCESS)
                e = cudaErrorUnknown;
        }
        if (e == cudaSuccess) e = cudaEventRecord(g_host.ev_b, g_host.copy);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, g_host.ev_b, 0);
        if (e != cudaSuccess) {
            // the kernel may be waiting on chunks that will never come: its watchdog releases it
            cudaStreamSynchronize(s);
            return cuda_fail(e, "streamed H2D copy");
        }
    }
    e = cudaMemcpyAsync(out_tokens, dTok, (size_t)B * T * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_num_tokens, dN, (size_t)B * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_scores, dS, (size_t)B * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && out_timestamps)
        e = cudaMemcpyAsync(out_timestamps, dTs, (size_t)B * T * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "decode_host copy/sync");
    // the device flags of this decode (length clamps, stream watchdog)
    uint32_t fl = 0;
    e = cudaMemcpy(&fl, (const char*)ws + wl.flags, sizeof(uint32_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "decode_host flags");
    if (out_flags) *out_flags = fl;
    if (fl & FLEXCTC_FLAG_STREAM_TIMEOUT)
        return fail(FLEXCTC_ERR_CUDA, "decode_host: a frame chunk never arrived (stream watchdog); outputs invalid");
    return FLEXCTC_OK;
}

}  // namespace
}  // namespace flexctc

extern "C" {

flexctc_status flexctc_decode_host(const float* log_probs_host, const int32_t* lengths_host, int32_t B, int32_t T,
                                   int32_t Vp1, const flexctc_config* cfg, const flexctc_lm* lm,
                                   const flexctc_boost* boost, void* device_scratch, size_t scratch_bytes,
                                   flexctc_stream stream, int32_t* out_tokens, int32_t* out_num_tokens,
                                   float* out_scores, int32_t* out_timestamps, uint32_t* out_flags) {
    return decode_host_impl(log_probs_host, false, lengths_host, B, T, Vp1, cfg, lm, boost, device_scratch,
                            scratch_bytes, stream, out_tokens, out_num_tokens, out_scores, out_timestamps, out_flags);
}

flexctc_status flexctc_decode_host_bf16(const uint16_t* logits_host, const int32_t* lengths_host, int32_t B, int32_t T,
                                        int32_t Vp1, const flexctc_config* cfg, const flexctc_lm* lm,
                                        const flexctc_boost* boost, void* device_scratch, size_t scratch_bytes,
                                        flexctc_stream stream, int32_t* out_tokens, int32_t* out_num_tokens,
                                        float* out_scores, int32_t* out_timestamps, uint32_t* out_flags) {
    return decode_host_impl(logits_host, true, lengths_host, B, T, Vp1, cfg, lm, boost, device_scratch,
                            scratch_bytes, stream, out_tokens, out_num_tokens, out_scores, out_timestamps, out_flags);
}

}  // extern "C"
