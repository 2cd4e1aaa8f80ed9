// ARPA -> "sorted-arc, state-indexed" n-gram LM layout (host side of flexctc_lm_load).
//
// Query semantics (NGPU-LM, §II-D, §III-B; standard backoff):
//   P(w | h) = p(h, w) if the n-gram (h, w) is listed, else bw(h) + P(w | h[1:]).
// A state is a listed context (an n-gram of order <= N-1, or the empty root context); the LM
// state of a hypothesis is the longest suffix of its history that is a state, so a
// query walks the backoff chain state -> bo(state) -> ... -> root accumulating bw in fp32 in
// that order (reading R19: identical order to the oracle's iteration from the longest history).
// The prefix property of ARPA files (every listed n-gram's context is itself listed) is
// required; it is what makes "first level with an arc" and "longest listed suffix" agree.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "flexctc_internal.h"

namespace flexctc {

namespace {

constexpr double kLn10 = 2.302585092994045684;  // log10 -> nats, rounded once to fp32 (R7)

struct KeyHash {
    size_t operator()(const std::string& s) const noexcept { return std::hash<std::string_view>()(s); }
};

inline std::string key_of(const int32_t* ids, int n) {
    return std::string(reinterpret_cast<const char*>(ids), sizeof(int32_t) * (size_t)n);
}

inline float f32_of(double log10v) { return (float)(log10v * kLn10); }

struct Gram {
    int n;
    int64_t ids_off;  // into ids
    double lp10, bw10;
    bool has_bw;
};

}  // namespace

flexctc_status build_lm_host(const char* path, int32_t V, const char* const* syms, LmHost& out) {
    if (V < 1) return fail(FLEXCTC_ERR_INVALID_ARG, "vocab_size must be >= 1");
    FILE* f = fopen(path, "rb");
    if (!f) return fail(FLEXCTC_ERR_IO, std::string("cannot open ") + path);
    std::string buf;
    {
        fseek(f, 0, SEEK_END);
        long sz = ftell(f);
        fseek(f, 0, SEEK_SET);
        if (sz < 0) { fclose(f); return fail(FLEXCTC_ERR_IO, std::string("cannot read ") + path); }
        buf.resize((size_t)sz);
        if (sz && fread(&buf[0], 1, (size_t)sz, f) != (size_t)sz) {
            fclose(f);
            return fail(FLEXCTC_ERR_IO, std::string("short read ") + path);
        }
        fclose(f);
    }

    std::unordered_map<std::string, int32_t> sym_id;
    std::vector<std::string> sym_name;
    std::vector<long> counts, seen;
    std::vector<Gram> grams;
    std::vector<int32_t> ids;
    int section = -1;
    bool ended = false;
    long lineno = 0;
    auto perr = [&](const std::string& m) {
        return fail(FLEXCTC_ERR_PARSE, std::string(path) + ":" + std::to_string(lineno) + ": " + m);
    };
    size_t pos = 0;
    std::vector<std::string_view> fs;
    while (pos < buf.size() && !ended) {
        size_t e = buf.find('\n', pos);
        if (e == std::string::npos) e = buf.size();
        std::string_view line(buf.data() + pos, e - pos);
        pos = e + 1;
        ++lineno;
        // split on blanks
        fs.clear();
        size_t i = 0;
        while (i < line.size()) {
            while (i < line.size() && (line[i] == ' ' || line[i] == '\t' || line[i] == '\r')) ++i;
            size_t j = i;
            while (j < line.size() && !(line[j] == ' ' || line[j] == '\t' || line[j] == '\r')) ++j;
            if (j > i) fs.emplace_back(line.data() + i, j - i);
            i = j;
        }
        if (fs.empty()) continue;
        if (fs[0] == "\\data\\") { section = 0; continue; }
        if (fs[0] == "\\end\\") { ended = true; break; }
        if (fs[0][0] == '\\') {
            std::string h(fs[0]);
            int n = 0;
            if (sscanf(h.c_str(), "\\%d-grams:", &n) != 1 || n < 1 || n > (int)counts.size())
                return perr("bad section header '" + h + "'");
            section = n;
            continue;
        }
        if (section == 0) {
            std::string h;
            for (auto& x : fs) { h += std::string(x); h += ' '; }
            int n;
            long c;
            if (sscanf(h.c_str(), "ngram %d=%ld", &n, &c) != 2 || n != (int)counts.size() + 1 || c < 0)
                return perr("bad count line");
            counts.push_back(c);
            seen.push_back(0);
            continue;
        }
        if (section < 1) return perr("text before \\data\\");
        const int n = section;
        if ((int)fs.size() != n + 1 && (int)fs.size() != n + 2) return perr("bad n-gram line");
        char tmp[64];
        auto num = [&](std::string_view s, double& v) {
            if (s.size() >= sizeof(tmp)) return false;
            memcpy(tmp, s.data(), s.size());
            tmp[s.size()] = 0;
            char* endp = nullptr;
            v = strtod(tmp, &endp);
            return *endp == 0;
        };
        Gram g{n, (int64_t)ids.size(), 0.0, 0.0, false};
        if (!num(fs[0], g.lp10)) return perr("bad log-prob");
        if ((int)fs.size() == n + 2) {
            if (!num(fs[n + 1], g.bw10)) return perr("bad backoff");
            g.has_bw = true;
        }
        for (int k = 1; k <= n; ++k) {
            std::string s(fs[k]);
            auto it = sym_id.find(s);
            int32_t id;
            if (it == sym_id.end()) {
                if (n > 1) return perr("n-gram references unseen symbol '" + s + "'");
                id = (int32_t)sym_name.size();
                sym_id.emplace(s, id);
                sym_name.push_back(s);
            } else {
                id = it->second;
            }
            ids.push_back(id);
        }
        grams.push_back(g);
        seen[n - 1]++;
    }
    if (!ended) return fail(FLEXCTC_ERR_PARSE, std::string(path) + ": missing \\end\\");
    for (size_t k = 0; k < counts.size(); ++k)
        if (counts[k] != seen[k])
            return fail(FLEXCTC_ERR_PARSE, std::string(path) + ": " + std::to_string(k + 1) + "-gram count mismatch");
    const int N = (int)counts.size();
    if (N < 1) return fail(FLEXCTC_ERR_PARSE, std::string(path) + ": no n-grams");
    auto find_sym = [&](const std::string& s) { auto it = sym_id.find(s); return it == sym_id.end() ? -1 : it->second; };
    const int BOS = find_sym("<s>"), EOS = find_sym("</s>"), UNK = find_sym("<unk>");
    if (EOS < 0) return fail(FLEXCTC_ERR_PARSE, std::string(path) + ": missing </s>");
    if (V > 65535) return fail(FLEXCTC_ERR_CAPACITY, "vocab_size > 65535");

    // decoder token <-> LM symbol binding (R7)
    std::vector<int32_t> tok2sym(V);
    std::vector<std::vector<int32_t>> sym2tok(sym_name.size());
    for (int w = 0; w < V; ++w) {
        std::string name = syms ? std::string(syms[w]) : std::to_string(w);
        int s = find_sym(name);
        if (s < 0) s = UNK;
        if (s < 0) return fail(FLEXCTC_ERR_VOCAB_BIND, "token '" + name + "' is not in the LM and there is no <unk>");
        tok2sym[w] = s;
        sym2tok[s].push_back(w);
    }

    // ---- states: root + every listed n-gram of order <= N-1 (prefix property checked)
    std::unordered_map<std::string, int32_t, KeyHash> state_of;
    state_of.reserve(grams.size());
    std::vector<int32_t> st_len{0};
    std::vector<int64_t> st_ids_off{0};
    std::vector<float> st_bw{0.0f};
    state_of.emplace(std::string(), 0);
    for (const Gram& g : grams) {
        if (g.n > N - 1) continue;
        auto r = state_of.emplace(key_of(&ids[g.ids_off], g.n), (int32_t)st_len.size());
        if (!r.second) return fail(FLEXCTC_ERR_PARSE, std::string(path) + ": duplicate n-gram");
        st_len.push_back(g.n);
        st_ids_off.push_back(g.ids_off);
        st_bw.push_back(g.has_bw ? f32_of(g.bw10) : 0.0f);
    }
    const int32_t S = (int32_t)st_len.size();
    auto state_ids = [&](int32_t s) { return &ids[st_ids_off[s]]; };
    // longest suffix of seq[0..n) (n <= N-1) that is a state
    auto longest_state_suffix = [&](const int32_t* seq, int n) -> int32_t {
        for (int l = n; l >= 1; --l) {
            auto it = state_of.find(key_of(seq + (n - l), l));
            if (it != state_of.end()) return it->second;
        }
        return 0;
    };
    std::vector<int32_t> st_bo(S, -1);
    for (int32_t s = 1; s < S; ++s) st_bo[s] = longest_state_suffix(state_ids(s) + 1, st_len[s] - 1);

    // ---- arcs (order >= 2) and the per-state </s> arc; the dense root row (order 1)
    struct Arc { int32_t s; int32_t tok; float lp; int32_t next; };
    std::vector<Arc> arcs;
    arcs.reserve(grams.size());
    std::vector<float> eos_arc(S, NAN);
    std::vector<uint8_t> has_eos(S, 0);
    std::vector<float> uni_sym(sym_name.size(), NAN);
    std::vector<int32_t> cat(N + 1);
    for (const Gram& g : grams) {
        const int32_t* gi = &ids[g.ids_off];
        const int32_t x = gi[g.n - 1];
        float lp = f32_of(g.lp10);
        int32_t ctx = 0;
        if (g.n > 1) {
            auto it = state_of.find(key_of(gi, g.n - 1));
            if (it == state_of.end()) {
                std::string ng;
                for (int k = 0; k < g.n; ++k) ng += (k ? " " : "") + sym_name[gi[k]];
                return fail(FLEXCTC_ERR_PARSE, std::string(path) + ": n-gram '" + ng + "' has an unlisted context");
            }
            ctx = it->second;
        } else {
            uni_sym[x] = lp;
        }
        if (x == EOS) { eos_arc[ctx] = lp; has_eos[ctx] = 1; }
        if (g.n == 1 || sym2tok[x].empty()) continue;
        // next state: longest state-suffix of (h + x), truncated to N-1 symbols
        int m = std::min(g.n, N - 1);
        int32_t next = longest_state_suffix(gi + (g.n - m), m);
        for (int32_t w : sym2tok[x]) arcs.push_back(Arc{ctx, w, lp, next});
    }
    if (!has_eos[0]) return fail(FLEXCTC_ERR_PARSE, std::string(path) + ": missing </s> unigram");
    std::sort(arcs.begin(), arcs.end(), [](const Arc& a, const Arc& b) { return a.s != b.s ? a.s < b.s : a.tok < b.tok; });

    out = LmHost();
    out.order = N;
    out.V = V;
    out.S = S;
    out.st_hdr.assign((size_t)S * 4, 0);
    out.arc_tok.resize(arcs.size());
    out.arc_val.resize(arcs.size() * 2);
    {
        size_t a = 0;
        for (int32_t s = 0; s < S; ++s) {
            size_t b = a;
            while (a < arcs.size() && arcs[a].s == s) ++a;
            int32_t* h = &out.st_hdr[(size_t)s * 4];
            h[0] = (int32_t)b;
            h[1] = (int32_t)(a - b);
            h[2] = st_bo[s];
            memcpy(&h[3], &st_bw[s], 4);
        }
        for (size_t k = 0; k < arcs.size(); ++k) {
            out.arc_tok[k] = (uint16_t)arcs[k].tok;
            memcpy(&out.arc_val[2 * k], &arcs[k].lp, 4);
            out.arc_val[2 * k + 1] = arcs[k].next;
        }
    }
    out.uni_lp.resize(V);
    out.uni_next.resize(V);
    for (int w = 0; w < V; ++w) {
        int32_t s = tok2sym[w];
        out.uni_lp[w] = uni_sym[s];
        out.uni_next[w] = N >= 2 ? longest_state_suffix(&s, 1) : 0;
    }
    // LM.Final per state: walk the chain accumulating bw in fp32 (R19)
    out.eos.resize(S);
    for (int32_t s = 0; s < S; ++s) {
        float acc = 0.0f;
        int32_t x = s;
        for (;;) {
            if (has_eos[x]) { out.eos[s] = acc + eos_arc[x]; break; }
            acc = acc + st_bw[x];
            x = st_bo[x];
        }
    }
    // pre-prune bound: ub(s) >= max_w log P(w | s) (fp64 recursion by context length + margin)
    {
        std::vector<double> ub(S, -INFINITY);
        double u0 = -INFINITY;
        for (int w = 0; w < V; ++w) u0 = std::max(u0, (double)out.uni_lp[w]);
        ub[0] = u0;
        std::vector<int32_t> ord(S);
        for (int32_t s = 0; s < S; ++s) ord[s] = s;
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return st_len[a] < st_len[b]; });
        for (int32_t s : ord) {
            if (s == 0) continue;
            const int32_t* h = &out.st_hdr[(size_t)s * 4];
            double m = (double)st_bw[s] + ub[st_bo[s]];
            for (int32_t k = h[0]; k < h[0] + h[1]; ++k) {
                float lp;
                memcpy(&lp, &out.arc_val[2 * k], 4);
                m = std::max(m, (double)lp);
            }
            ub[s] = m;
        }
        out.ub.resize(S);
        for (int32_t s = 0; s < S; ++s) out.ub[s] = (float)(ub[s] + 1e-5 * (1.0 + std::fabs(ub[s])));
    }
    out.start = (BOS >= 0 && N >= 2) ? longest_state_suffix(&BOS, 1) : 0;

    // ---- device query structures:
    // per-state record = the whole backoff chain unrolled: arc levels (contexts of length >= 2:
    // CSR offset, degree, and the fp32 backoff sum accumulated when the sequential walk reaches
    // that level), the length-1 context (index of its dense row) with its accumulated sum, the
    // sum at the root, the pre-prune bound and LM.Final. All levels can then be searched in
    // parallel and the first level holding the token wins — bit-identical to the sequential walk.
    out.NL = std::max(0, N - 2);
    out.RW = ((8 + 3 * out.NL) + 3) & ~3;
    std::vector<int32_t> dense_idx(S, -1);
    int32_t U = 0;
    for (int32_t s = 1; s < S; ++s)
        if (st_len[s] == 1) dense_idx[s] = U++;
    out.U = U;
    out.rec.assign((size_t)S * out.RW, 0);
    for (int32_t s = 0; s < S; ++s) {
        int32_t* r = &out.rec[(size_t)s * out.RW];
        float acc = 0.0f, cum_u = 0.0f;
        int32_t x = s, n = 0, u = -1;
        while (x != 0) {
            if (st_len[x] >= 2) {
                const int32_t* h = &out.st_hdr[(size_t)x * 4];
                r[8 + 3 * n] = h[0];
                r[8 + 3 * n + 1] = h[1];
                memcpy(&r[8 + 3 * n + 2], &acc, 4);
                ++n;
            } else {
                u = dense_idx[x];
                cum_u = acc;
            }
            acc = acc + st_bw[x];
            x = st_bo[x];
        }
        // token signature of the arc levels: bit sig_bit(w) is set for every token with an arc
        // at one of them, so a query whose bit is clear goes straight to the dense / root level
        uint64_t sig = 0;
        for (int j = 0; j < n; ++j)
            for (int32_t k = r[8 + 3 * j]; k < r[8 + 3 * j] + r[8 + 3 * j + 1]; ++k)
                sig |= 1ull << lm_sig_bit(out.arc_tok[k]);
        memcpy(&r[6], &sig, 8);
        r[0] = n;
        r[1] = u;
        memcpy(&r[2], &cum_u, 4);
        memcpy(&r[3], &acc, 4);
        memcpy(&r[4], &out.ub[s], 4);
        memcpy(&r[5], &out.eos[s], 4);
    }
    // dense rows of the length-1 contexts: {value, next | found<<31} for every decoder token
    out.dense.assign((size_t)U * V * 2, 0);
    for (int32_t s = 1; s < S; ++s) {
        if (dense_idx[s] < 0) continue;
        const int32_t* h = &out.st_hdr[(size_t)s * 4];
        int32_t* row = &out.dense[(size_t)dense_idx[s] * V * 2];
        for (int w = 0; w < V; ++w) {
            float v = out.uni_lp[w];
            int32_t nx = out.uni_next[w];
            const uint16_t* b = out.arc_tok.data() + h[0];
            const uint16_t* e = b + h[1];
            const uint16_t* it = std::lower_bound(b, e, (uint16_t)w);
            if (it != e && *it == (uint16_t)w) {
                size_t k = (size_t)(it - out.arc_tok.data());
                memcpy(&v, &out.arc_val[2 * k], 4);
                nx = out.arc_val[2 * k + 1] | (int32_t)0x80000000u;
            }
            memcpy(&row[2 * w], &v, 4);
            row[2 * w + 1] = nx;
        }
    }
    return FLEXCTC_OK;
}

// Host mirror of the device query (beam_kernel.cu lm_query): the same record walk, the same
// fp32 operations in the same order.
float lm_query_host(const LmHost& lm, int32_t s, int32_t w, int32_t* next) {
    const int32_t* r = &lm.rec[(size_t)s * lm.RW];
    for (int j = 0; j < r[0]; ++j) {
        const uint16_t* b = lm.arc_tok.data() + r[8 + 3 * j];
        const uint16_t* e = b + r[8 + 3 * j + 1];
        const uint16_t* it = std::lower_bound(b, e, (uint16_t)w);
        if (it != e && *it == (uint16_t)w) {
            size_t k = (size_t)(it - lm.arc_tok.data());
            float lp, cum;
            memcpy(&lp, &lm.arc_val[2 * k], 4);
            memcpy(&cum, &r[8 + 3 * j + 2], 4);
            *next = lm.arc_val[2 * k + 1];
            return cum + lp;
        }
    }
    float cum_u, cum_root;
    memcpy(&cum_u, &r[2], 4);
    memcpy(&cum_root, &r[3], 4);
    if (r[1] >= 0) {
        const int32_t* d = &lm.dense[((size_t)r[1] * lm.V + w) * 2];
        float v;
        memcpy(&v, &d[0], 4);
        const bool found = (d[1] & (int32_t)0x80000000u) != 0;
        *next = d[1] & 0x7fffffff;
        return (found ? cum_u : cum_root) + v;
    }
    *next = lm.uni_next[w];
    return cum_root + lm.uni_lp[w];
}

}  // namespace flexctc
