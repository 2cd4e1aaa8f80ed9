// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h). Plain loops, one utterance at a time,
// independent representations: a hypothesis is a token tuple (no hashes), the LM is a direct
// ARPA backoff evaluator over the full history (no state machine), the booster is naive
// suffix matching over the phrase set (no failure links).
//
// Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n; Rn = DESIGN.md reading n.
// Build: g++ -O2 -std=c++17 -ffp-contract=off (no fast-math, no FMA contraction: R19).
#include "oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

thread_local std::string g_err;
void set_err(const std::string& s) { g_err = s; }

struct VecHash {
    size_t operator()(const std::vector<int>& v) const {
        size_t h = 1469598103934665603ull;
        for (int x : v) { h ^= (size_t)(uint32_t)x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2); }
        return h;
    }
};

// fl32 / fl64 fused multiply-add (explicit: the only contraction the canonical order allows, R19)
inline float fma_r(float a, float b, float c) { return fmaf(a, b, c); }
inline double fma_r(double a, double b, double c) { return fma(a, b, c); }

// ======================================================================================
// LM: ARPA parse + direct backoff recursion (semantics S:170-198; R7)
// ======================================================================================
struct Arpa {
    int order = 0;
    std::unordered_map<std::string, int> sym;
    std::vector<std::string> names;
    int bos = -1, eos = -1, unk = -1;
    struct E { double lp; double bw; };  // nats; bw = 0 when the file gives none
    std::unordered_map<std::vector<int>, E, VecHash> grams;
    std::vector<int> tok2sym;             // decoder token -> LM symbol (R7)
};

std::vector<std::string> split_ws(const std::string& s) {
    std::vector<std::string> out;
    std::istringstream is(s);
    std::string w;
    while (is >> w) out.push_back(w);
    return out;
}

Arpa* parse_arpa(const char* path, int V, const char* const* token_symbols) {
    std::ifstream f(path);
    if (!f) { set_err(std::string("cannot open ") + path); return nullptr; }
    auto* a = new Arpa();
    std::string line;
    int lineno = 0;
    std::vector<long> counts;
    int section = -1;  // -1 before \data\, 0 in \data\, n in \n-grams:
    bool ended = false;
    std::vector<long> seen;
    auto fail = [&](const std::string& m) { set_err(std::string(path) + ":" + std::to_string(lineno) + ": " + m); delete a; return (Arpa*)nullptr; };
    const double LN10 = 2.302585092994045684;  // ln 10 (log10 -> natural log)
    while (std::getline(f, line)) {
        ++lineno;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        std::string t = line;
        size_t b = t.find_first_not_of(" \t");
        if (b == std::string::npos) continue;
        t = t.substr(b);
        if (t == "\\data\\") { section = 0; continue; }
        if (t == "\\end\\") { ended = true; break; }
        if (t[0] == '\\') {
            int n = 0;
            if (sscanf(t.c_str(), "\\%d-grams:", &n) != 1 || n < 1 || n > (int)counts.size())
                return fail("bad section header '" + t + "'");
            section = n;
            continue;
        }
        if (section == 0) {
            int n; long c;
            if (sscanf(t.c_str(), "ngram %d=%ld", &n, &c) != 2 || n != (int)counts.size() + 1)
                return fail("bad count line");
            counts.push_back(c);
            seen.push_back(0);
            continue;
        }
        if (section < 1) return fail("text before \\data\\");
        std::vector<std::string> fs = split_ws(t);
        int n = section;
        if ((int)fs.size() != n + 1 && (int)fs.size() != n + 2) return fail("bad n-gram line");
        char* end = nullptr;
        double lp10 = strtod(fs[0].c_str(), &end);
        if (*end) return fail("bad log-prob");
        double bw10 = 0.0;
        if ((int)fs.size() == n + 2) {
            bw10 = strtod(fs[n + 1].c_str(), &end);
            if (*end) return fail("bad backoff");
        }
        std::vector<int> key;
        for (int i = 1; i <= n; ++i) {
            auto it = a->sym.find(fs[i]);
            int id;
            if (it == a->sym.end()) {
                if (n > 1) return fail("n-gram references unseen symbol '" + fs[i] + "'");
                id = (int)a->names.size();
                a->sym[fs[i]] = id;
                a->names.push_back(fs[i]);
            } else {
                id = it->second;
            }
            key.push_back(id);
        }
        a->grams[key] = Arpa::E{lp10 * LN10, bw10 * LN10};
        seen[n - 1]++;
    }
    if (!ended) return fail("missing \\end\\");
    for (size_t i = 0; i < counts.size(); ++i)
        if (counts[i] != seen[i]) return fail(std::to_string(i + 1) + "-gram count mismatch");
    a->order = (int)counts.size();
    auto g = [&](const char* s) { auto it = a->sym.find(s); return it == a->sym.end() ? -1 : it->second; };
    a->bos = g("<s>");
    a->eos = g("</s>");
    a->unk = g("<unk>");
    if (a->eos < 0) return fail("missing </s>");  // Alg. 1 needs LM.Final
    a->tok2sym.resize(V);
    for (int w = 0; w < V; ++w) {
        std::string name = token_symbols ? std::string(token_symbols[w]) : std::to_string(w);
        int s = g(name.c_str());
        if (s < 0) s = a->unk;
        if (s < 0) { set_err("token '" + name + "' not in LM and no <unk>"); delete a; return nullptr; }
        a->tok2sym[w] = s;
    }
    return a;
}

// log P(w | hist) by the standard backoff recursion, iterated from the longest history to
// the shortest: acc = 0; for h = last N-1 tokens down to (): if (h,w) listed
// return acc + p(h,w); else acc += bw(h) (0 when h is unlisted or has no backoff).
template <class R>
R lm_logp_sym(const Arpa& a, const std::vector<int>& hist, int wsym) {
    R acc = 0;
    int hl = std::min((int)hist.size(), a.order - 1);
    for (int len = hl; len >= 0; --len) {
        std::vector<int> key(hist.end() - len, hist.end());
        key.push_back(wsym);
        auto it = a.grams.find(key);
        if (it != a.grams.end()) return acc + (R)it->second.lp;
        if (len > 0) {
            key.pop_back();
            auto ic = a.grams.find(key);
            if (ic != a.grams.end()) acc = acc + (R)ic->second.bw;
        }
    }
    // unreachable for symbols that have a unigram
    return -std::numeric_limits<R>::infinity();
}

// History seen by the LM for a decoder prefix: <s> followed by the mapped tokens (P:116 LM(<SOS>)).
std::vector<int> lm_history(const Arpa& a, const std::vector<int>& prefix) {
    std::vector<int> h;
    if (a.bos >= 0) h.push_back(a.bos);  // no <s> -> empty context
    for (int w : prefix) h.push_back(a.tok2sym[w]);
    return h;
}

// ======================================================================================
// Boosting: naive suffix matching over the phrase set (reward law S:263-275, R17)
// ======================================================================================
struct Boost {
    double w = 1.0;
    int maxlen = 0;
    std::set<std::vector<int>> phrases;
    std::set<std::vector<int>> prefixes;  // every prefix of every phrase, including ()
};

// state(p) = the longest suffix of p that is a prefix of some phrase (string comparison)
std::vector<int> bt_state(const Boost& bt, const std::vector<int>& p) {
    int n = (int)p.size();
    for (int len = std::min(n, bt.maxlen); len >= 0; --len) {
        std::vector<int> s(p.end() - len, p.end());
        if (bt.prefixes.count(s)) return s;
    }
    return {};
}

template <class R> R bt_C(const Boost& bt, int depth) { return (R)bt.w * (R)depth; }  // C = w·depth

// committed(v) = C(deepest final ancestor-or-self); pcom(v) = C(deepest final strict ancestor)
template <class R> R bt_committed(const Boost& bt, const std::vector<int>& v, bool strict) {
    for (int len = (int)v.size() - (strict ? 1 : 0); len >= 1; --len) {
        std::vector<int> pre(v.begin(), v.begin() + len);
        if (bt.phrases.count(pre)) return bt_C<R>(bt, len);
    }
    return 0;
}
template <class R> R bt_U(const Boost& bt, const std::vector<int>& v) {  // U = C - committed
    return bt_C<R>(bt, (int)v.size()) - bt_committed<R>(bt, v, false);
}
template <class R> R bt_dC(const Boost& bt, const std::vector<int>& v) {  // ΔC at final nodes
    if (!bt.phrases.count(v)) return 0;
    return bt_C<R>(bt, (int)v.size()) - bt_committed<R>(bt, v, true);
}
// delta(u, a) = ΔC(v) + U(v) - U(u) with v = δ(u, a)
template <class R> R bt_delta(const Boost& bt, const std::vector<int>& prefix, int w) {
    std::vector<int> u = bt_state(bt, prefix);
    std::vector<int> pw = prefix;
    pw.push_back(w);
    std::vector<int> v = bt_state(bt, pw);
    R g = bt_dC<R>(bt, v) + bt_U<R>(bt, v);
    return g - bt_U<R>(bt, u);
}

// ======================================================================================
// Decoder: Algorithm 1, one utterance, step order of SPEC S:349-358
// ======================================================================================
template <class R>
struct Hyp {
    std::vector<int> prefix;  // collapsed transcript ("merging repeated labels and removing blanks")
    int last;                 // beams.last_labels
    R score;                  // acc_scores
    std::vector<int> align;   // frame labels ("token and pointer tensors")
    bool alive;
};

template <class R> struct Cand { R s; long f; };

template <class R>
struct Ctx {
    const oracle_cfg* cfg;
    const Arpa* lm;
    const Boost* bt;
    int V;  // non-blank vocabulary
    // memoised pure functions of the (N-1)-token LM history / maxlen-token boost history
    std::unordered_map<std::vector<int>, std::vector<R>, VecHash> lm_rows, bt_rows;

    const std::vector<R>& lm_row(const std::vector<int>& prefix) {  // [V] logp + [V] = final
        std::vector<int> h = lm_history(*lm, prefix);
        std::vector<int> key(h.end() - std::min((int)h.size(), lm->order - 1), h.end());
        auto it = lm_rows.find(key);
        if (it != lm_rows.end()) return it->second;
        std::vector<R> row(V + 1);
        for (int w = 0; w < V; ++w) row[w] = lm_logp_sym<R>(*lm, key, lm->tok2sym[w]);
        row[V] = lm_logp_sym<R>(*lm, key, lm->eos);
        return lm_rows.emplace(key, std::move(row)).first->second;
    }
    const std::vector<R>& bt_row(const std::vector<int>& prefix) {  // [V] deltas + [V] = U(state)
        std::vector<int> key(prefix.end() - std::min((int)prefix.size(), bt->maxlen), prefix.end());
        auto it = bt_rows.find(key);
        if (it != bt_rows.end()) return it->second;
        std::vector<R> row(V + 1);
        for (int w = 0; w < V; ++w) row[w] = bt_delta<R>(*bt, key, w);
        row[V] = bt_U<R>(*bt, bt_state(*bt, key));
        return bt_rows.emplace(key, std::move(row)).first->second;
    }
};

// Canonical combiner for a merge group already ordered by (score desc, slot asc)  (R13, R14):
// s0 + log1p(Σ_{i>=1, in order} exp(s_i - s0)); exp/log1p evaluated in fp64 then rounded.
template <class R> R combine(const std::vector<R>& s, int merge_mode) {
    R s0 = s[0];
    if (merge_mode == 1) return s0;
    R sum = 0;
    for (size_t i = 1; i < s.size(); ++i) {
        R d = s[i] - s0;
        sum = sum + (R)std::exp((double)d);
    }
    return s0 + (R)std::log1p((double)sum);
}

struct UttOut {
    std::vector<int> tokens, timestamps, align;
    double score;
};

template <class R>
std::vector<std::pair<Hyp<R>, int>> decode_utt(const std::vector<std::vector<R>>& D, int Vp1, int L,
                                               const oracle_cfg* cfg, const Arpa* lm, const Boost* bt) {
    const R NEG = -std::numeric_limits<R>::infinity();
    const int K = cfg->beam;
    const int blank = Vp1 - 1;  // R1: blank = last index
    const R alpha_lm = (R)cfg->alpha_lm, alpha_bt = (R)cfg->alpha_bt, beta = (R)cfg->beta;
    const R theta = (R)cfg->theta;
    Ctx<R> ctx{cfg, lm, bt, Vp1 - 1, {}, {}};

    // init: slot 0 score 0, others -inf; last = blank (R6); LM at <s>; BT at root
    std::vector<Hyp<R>> slots(K);
    for (int k = 0; k < K; ++k) slots[k] = Hyp<R>{{}, blank, k == 0 ? (R)0 : NEG, {}, k == 0};

    std::vector<Cand<R>> cand((size_t)K * Vp1);
    for (int t = 0; t < L; ++t) {  // t >= L: row frozen (R16)
        const std::vector<R>& Dt = D[t];
        // candidate scores, Eq. (1) / Alg. 1, canonical order (R19)
        for (int k = 0; k < K; ++k) {
            const Hyp<R>& h = slots[k];
            const std::vector<R>* lr = (h.alive && lm) ? &ctx.lm_row(h.prefix) : nullptr;
            const std::vector<R>* br = (h.alive && bt) ? &ctx.bt_row(h.prefix) : nullptr;
            for (int w = 0; w < Vp1; ++w) {
                long f = (long)k * Vp1 + w;
                R s = NEG;
                if (h.alive) {
                    s = h.score + Dt[w];                     // logp <- D[:,t,:] + acc
                    if (w != blank && w != h.last) {         // ¬rb_mask (R2)
                        s = s + beta;                        // P:127 (R8)
                        if (lm) s = fma_r(alpha_lm, (*lr)[w], s);
                        if (bt) s = fma_r(alpha_bt, (*br)[w], s);
                    } else if (cfg->fuse_repeats && w != blank) {
                        // P:167 variant: the repeated emission is scored by the LM / BT at each
                        // occurrence (no β, no state advance: the prefix is unchanged)
                        if (lm) s = fma_r(alpha_lm, (*lr)[w], s);
                        if (bt) s = fma_r(alpha_bt, (*br)[w], s);
                    }
                }
                cand[f] = Cand<R>{s, f};
            }
        }
        if (cfg->merge_first) {
            // Reading R27 (BJ north_star: "merges duplicate prefixes by prefix hash, selects the
            // top-K"): every candidate is first combined with the candidates of the same
            // (transcript, last label) (R12) by the R13/R14 combiner, members ordered by (score
            // desc, flat index asc); the K best groups by (merged score desc, flat index of the
            // group's best member asc) are kept (R9's tie rule on the representative), then the
            // θ-prune relative to the best group. The best member is the survivor:
            // its slot and label give the backpointer and the alignment.
            std::map<std::pair<std::vector<int>, int>, std::vector<Cand<R>>> groups;
            for (const Cand<R>& c : cand) {  // flat index order
                if (c.s == NEG) continue;
                const int k = (int)(c.f / Vp1), w = (int)(c.f % Vp1);
                std::vector<int> pre = slots[k].prefix;
                if (w != blank && w != slots[k].last) pre.push_back(w);
                groups[{std::move(pre), w}].push_back(c);
            }
            std::vector<Cand<R>> gl;  // {merged score, flat index of the best member}
            for (auto& kv : groups) {
                std::vector<Cand<R>>& g = kv.second;
                std::stable_sort(g.begin(), g.end(), [](const Cand<R>& a, const Cand<R>& b) { return a.s > b.s; });
                std::vector<R> sc;
                for (const Cand<R>& c : g) sc.push_back(c.s);
                gl.push_back(Cand<R>{combine<R>(sc, cfg->merge_mode), g[0].f});
            }
            std::sort(gl.begin(), gl.end(), [](const Cand<R>& a, const Cand<R>& b) {
                if (a.s != b.s) return a.s > b.s;
                return a.f < b.f;
            });
            std::vector<Hyp<R>> nxt(K);
            const R gthr = gl.empty() ? NEG : gl[0].s - theta;
            for (int i = 0; i < K; ++i) {
                if (i >= (int)gl.size() || gl[i].s < gthr) { nxt[i] = Hyp<R>{{}, blank, NEG, {}, false}; continue; }
                const int k = (int)(gl[i].f / Vp1), w = (int)(gl[i].f % Vp1);
                const Hyp<R>& p = slots[k];
                Hyp<R> h;
                h.prefix = p.prefix;
                if (w != blank && w != p.last) h.prefix.push_back(w);
                h.last = w;
                h.score = gl[i].s;
                h.align = p.align;
                h.align.push_back(w);
                h.alive = true;
                nxt[i] = std::move(h);
            }
            slots = std::move(nxt);
            continue;
        }
        // flat TopK, ties -> lower flat index (R9)
        std::partial_sort(cand.begin(), cand.begin() + K, cand.end(), [](const Cand<R>& a, const Cand<R>& b) {
            if (a.s != b.s) return a.s > b.s;
            return a.f < b.f;
        });
        R mx = cand[0].s;                  // max_score
        R thr = mx - theta;                // acc < max - θ -> -inf (R10)
        std::vector<Hyp<R>> nxt(K);
        for (int i = 0; i < K; ++i) {
            const Cand<R>& c = cand[i];
            if (c.s == NEG || c.s < thr) { nxt[i] = Hyp<R>{{}, blank, NEG, {}, false}; continue; }
            int k = (int)(c.f / Vp1), w = (int)(c.f % Vp1);  // new_beamid, new_labels
            const Hyp<R>& p = slots[k];
            Hyp<R> h;
            h.prefix = p.prefix;
            if (w != blank && w != p.last) h.prefix.push_back(w);  // state/hash advance only on emission (R5)
            h.last = w;
            h.score = c.s;
            h.align = p.align;
            h.align.push_back(w);
            h.alive = true;
            nxt[i] = std::move(h);
        }
        // RecombineHypotheses: key (transcript, last label) (R12), survivor = best (score desc, slot asc)
        std::map<std::pair<std::vector<int>, int>, std::vector<int>> groups;
        for (int i = 0; i < K; ++i)
            if (nxt[i].alive) groups[{nxt[i].prefix, nxt[i].last}].push_back(i);
        for (auto& kv : groups) {
            std::vector<int>& g = kv.second;
            if (g.size() < 2) continue;
            std::stable_sort(g.begin(), g.end(), [&](int x, int y) {
                if (nxt[x].score != nxt[y].score) return nxt[x].score > nxt[y].score;
                return x < y;
            });
            std::vector<R> sc;
            for (int i : g) sc.push_back(nxt[i].score);
            nxt[g[0]].score = combine<R>(sc, cfg->merge_mode);
            for (size_t j = 1; j < g.size(); ++j) { nxt[g[j]].alive = false; nxt[g[j]].score = NEG; }
        }
        slots = std::move(nxt);
    }
    // EOS: beams.scores += α_LM · LM.Final(lm_sts)
    for (int k = 0; k < K; ++k) {
        Hyp<R>& h = slots[k];
        if (!h.alive) continue;
        if (lm) h.score = fma_r(alpha_lm, ctx.lm_row(h.prefix)[Vp1 - 1], h.score);
        if (bt && cfg->retract_boost_at_eos) h.score = fma_r(-alpha_bt, ctx.bt_row(h.prefix)[Vp1 - 1], h.score);
    }
    // final merge by transcript across last labels (R15), then order by (score desc, slot asc)
    std::map<std::vector<int>, std::vector<int>> groups;
    for (int k = 0; k < K; ++k)
        if (slots[k].alive) groups[slots[k].prefix].push_back(k);
    std::vector<std::pair<Hyp<R>, int>> out;
    for (auto& kv : groups) {
        std::vector<int>& g = kv.second;
        std::stable_sort(g.begin(), g.end(), [&](int x, int y) {
            if (slots[x].score != slots[y].score) return slots[x].score > slots[y].score;
            return x < y;
        });
        std::vector<R> sc;
        for (int i : g) sc.push_back(slots[i].score);
        Hyp<R> h = slots[g[0]];
        h.score = combine<R>(sc, cfg->merge_mode);
        out.emplace_back(std::move(h), g[0]);
    }
    std::stable_sort(out.begin(), out.end(), [](const std::pair<Hyp<R>, int>& a, const std::pair<Hyp<R>, int>& b) {
        if (a.first.score != b.first.score) return a.first.score > b.first.score;
        return a.second < b.second;
    });
    return out;
}

// timestamps (R20): frame where each token of the survivor's alignment was emitted
std::vector<int> emission_frames(const std::vector<int>& align, int blank) {
    std::vector<int> ts;
    int prev = blank;
    for (int t = 0; t < (int)align.size(); ++t) {
        int w = align[t];
        if (w != blank && w != prev) ts.push_back(t);
        prev = w;
    }
    return ts;
}

bool check_cfg(const oracle_cfg* cfg) {
    if (!cfg || cfg->beam < 1) { set_err("beam must be >= 1"); return false; }
    if (!(cfg->theta >= 0)) { set_err("theta must be >= 0"); return false; }
    return true;
}

}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

void* oracle_lm_load(const char* arpa_path, int32_t vocab_size, const char* const* token_symbols) {
    return parse_arpa(arpa_path, vocab_size, token_symbols);
}
void oracle_lm_free(void* lm) { delete (Arpa*)lm; }
int32_t oracle_lm_order(const void* lm) { return ((const Arpa*)lm)->order; }

double oracle_lm_logp(const void* lmv, const int32_t* hist, int32_t n, int32_t w, int32_t f32) {
    const Arpa& a = *(const Arpa*)lmv;
    std::vector<int> prefix(hist, hist + n);
    std::vector<int> h = lm_history(a, prefix);
    int ws = w < 0 ? a.eos : a.tok2sym[w];
    return f32 ? (double)lm_logp_sym<float>(a, h, ws) : lm_logp_sym<double>(a, h, ws);
}

// log P(w | hist) for many tokens after one history (the same evaluator as oracle_lm_logp)
void oracle_lm_logp_many(const void* lmv, const int32_t* hist, int32_t n, const int32_t* ws, int32_t m, int32_t f32,
                         double* out) {
    const Arpa& a = *(const Arpa*)lmv;
    std::vector<int> prefix(hist, hist + n);
    std::vector<int> h = lm_history(a, prefix);
    for (int32_t i = 0; i < m; ++i) {
        int wsym = ws[i] < 0 ? a.eos : a.tok2sym[ws[i]];
        out[i] = f32 ? (double)lm_logp_sym<float>(a, h, wsym) : lm_logp_sym<double>(a, h, wsym);
    }
}

double oracle_lm_seq(const void* lmv, const int32_t* toks, int32_t n) {
    const Arpa& a = *(const Arpa*)lmv;
    double s = 0;
    std::vector<int> prefix;
    for (int i = 0; i < n; ++i) {
        s += lm_logp_sym<double>(a, lm_history(a, prefix), a.tok2sym[toks[i]]);
        prefix.push_back(toks[i]);
    }
    return s + lm_logp_sym<double>(a, lm_history(a, prefix), a.eos);
}

void* oracle_boost_build(const int32_t* tokens, const int64_t* offsets, int32_t n_phrases,
                         double token_weight, int32_t vocab_size) {
    if (n_phrases <= 0) { set_err("empty phrase list"); return nullptr; }
    if (!(token_weight > 0)) { set_err("token_weight must be > 0"); return nullptr; }
    auto* bt = new Boost();
    bt->w = token_weight;
    for (int i = 0; i < n_phrases; ++i) {
        int64_t b = offsets[i], e = offsets[i + 1];
        if (e <= b) { set_err("empty phrase " + std::to_string(i)); delete bt; return nullptr; }
        std::vector<int> ph;
        for (int64_t j = b; j < e; ++j) {
            if (tokens[j] < 0 || tokens[j] >= vocab_size) {  // blank (= vocab_size) or out of range
                set_err("phrase " + std::to_string(i) + " has token out of [0, V)");
                delete bt;
                return nullptr;
            }
            ph.push_back(tokens[j]);
        }
        bt->maxlen = std::max(bt->maxlen, (int)ph.size());
        for (size_t l = 0; l <= ph.size(); ++l) bt->prefixes.insert(std::vector<int>(ph.begin(), ph.begin() + l));
        bt->phrases.insert(ph);
    }
    return bt;
}
void oracle_boost_free(void* bt) { delete (Boost*)bt; }

double oracle_boost_delta(const void* btv, const int32_t* prefix, int32_t n, int32_t w, int32_t f32) {
    const Boost& bt = *(const Boost*)btv;
    std::vector<int> p(prefix, prefix + n);
    return f32 ? (double)bt_delta<float>(bt, p, w) : bt_delta<double>(bt, p, w);
}
double oracle_boost_U(const void* btv, const int32_t* prefix, int32_t n, int32_t f32) {
    const Boost& bt = *(const Boost*)btv;
    std::vector<int> s = bt_state(bt, std::vector<int>(prefix, prefix + n));
    return f32 ? (double)bt_U<float>(bt, s) : bt_U<double>(bt, s);
}
int32_t oracle_boost_state_depth(const void* btv, const int32_t* prefix, int32_t n) {
    const Boost& bt = *(const Boost*)btv;
    return (int32_t)bt_state(bt, std::vector<int>(prefix, prefix + n)).size();
}

int32_t oracle_decode_f32(const float* log_probs, int64_t stride_b, int64_t stride_t,
                          const int32_t* lengths, int32_t B, int32_t T, int32_t Vp1,
                          const oracle_cfg* cfg, const void* lm, const void* bt, int32_t nthreads,
                          int32_t* out_tokens, int32_t* out_num_tokens, float* out_scores,
                          int32_t* out_timestamps, int32_t* out_alignment) {
    if (!check_cfg(cfg)) return 1;
    if (Vp1 < 2 || B < 0 || T < 0) { set_err("bad shape"); return 1; }
    std::atomic<int> next{0};
    auto work = [&]() {
        for (;;) {
            int b = next.fetch_add(1);
            if (b >= B) return;
            int L = std::max(0, std::min((int)lengths[b], (int)T));
            std::vector<std::vector<float>> D(L, std::vector<float>(Vp1));
            for (int t = 0; t < L; ++t)
                for (int w = 0; w < Vp1; ++w) D[t][w] = log_probs[b * stride_b + t * stride_t + w];
            auto res = decode_utt<float>(D, Vp1, L, cfg, (const Arpa*)lm, (const Boost*)bt);
            int32_t* tok = out_tokens + (int64_t)b * T;
            int32_t* ts = out_timestamps ? out_timestamps + (int64_t)b * T : nullptr;
            int32_t* al = out_alignment ? out_alignment + (int64_t)b * T : nullptr;
            for (int t = 0; t < T; ++t) { tok[t] = -1; if (ts) ts[t] = -1; if (al) al[t] = -1; }
            if (res.empty()) {  // every slot dead (only possible when D is -inf everywhere)
                out_num_tokens[b] = 0;
                out_scores[b] = -std::numeric_limits<float>::infinity();
                continue;
            }
            const Hyp<float>& h = res[0].first;
            std::vector<int> fr = emission_frames(h.align, Vp1 - 1);
            out_num_tokens[b] = (int)h.prefix.size();
            out_scores[b] = h.score;
            for (size_t i = 0; i < h.prefix.size(); ++i) { tok[i] = h.prefix[i]; if (ts) ts[i] = fr[i]; }
            if (al) for (size_t t = 0; t < h.align.size(); ++t) al[t] = h.align[t];
        }
    };
    int nt = std::max(1, nthreads);
    std::vector<std::thread> th;
    for (int i = 1; i < nt; ++i) th.emplace_back(work);
    work();
    for (auto& x : th) x.join();
    return 0;
}

int32_t oracle_decode_nbest(const double* log_probs, int32_t T, int32_t Vp1, int32_t L,
                            const oracle_cfg* cfg, const void* lm, const void* bt, int32_t f32,
                            int32_t max_out, int32_t* tokens_out, int32_t* lens_out,
                            double* scores_out) {
    if (!check_cfg(cfg)) return -1;
    L = std::max(0, std::min(L, T));
    auto emit = [&](auto res) {
        int n = std::min((int)res.size(), (int)max_out);
        for (int i = 0; i < n; ++i) {
            const auto& h = res[i].first;
            lens_out[i] = (int)h.prefix.size();
            for (int t = 0; t < T; ++t) tokens_out[(int64_t)i * T + t] = t < (int)h.prefix.size() ? h.prefix[t] : -1;
            scores_out[i] = (double)h.score;
        }
        return (int32_t)res.size();
    };
    if (f32) {
        std::vector<std::vector<float>> D(L, std::vector<float>(Vp1));
        for (int t = 0; t < L; ++t) for (int w = 0; w < Vp1; ++w) D[t][w] = (float)log_probs[(int64_t)t * Vp1 + w];
        return emit(decode_utt<float>(D, Vp1, L, cfg, (const Arpa*)lm, (const Boost*)bt));
    }
    std::vector<std::vector<double>> D(L, std::vector<double>(Vp1));
    for (int t = 0; t < L; ++t) for (int w = 0; w < Vp1; ++w) D[t][w] = log_probs[(int64_t)t * Vp1 + w];
    return emit(decode_utt<double>(D, Vp1, L, cfg, (const Arpa*)lm, (const Boost*)bt));
}

// log-softmax of bf16 logits, the plain definition (R25): bf16 -> its exact value (the upper 16
// bits of an fp32), max, fp64 sum of exp in index order, lse, one rounding per output
int32_t oracle_log_softmax_bf16(const uint16_t* x, int64_t n_rows, int64_t stride, int32_t Vp1, float* out) {
    for (int64_t i = 0; i < n_rows; ++i) {
        std::vector<double> v(Vp1);
        for (int w = 0; w < Vp1; ++w) {
            uint32_t bits = (uint32_t)x[i * stride + w] << 16;
            float f;
            std::memcpy(&f, &bits, 4);
            v[w] = (double)f;
        }
        double m = v[0];
        for (int w = 1; w < Vp1; ++w) m = std::max(m, v[w]);
        double S = 0.0;
        for (int w = 0; w < Vp1; ++w) S += std::exp(v[w] - m);
        const double lse = m + std::log(S);
        for (int w = 0; w < Vp1; ++w) out[i * Vp1 + w] = (float)(v[w] - lse);
    }
    return 0;
}

}  // extern "C"
