// Phrases -> Aho-Corasick boosting automaton with a dense transition table (host side of
// flexctc_boost_build).
//
// GPU-PB (§III-B): "a phrase prefix tree—constructed using the Aho-Corasick
// algorithm ... progressively distributes boosting scores along the prefix tree based on node
// depth". The concrete reward law is reading R17:
//   C(n) = w·depth(n), committed(n) = C(deepest final ancestor-or-self), U = C - committed,
//   pcom(n) = C(deepest final strict ancestor), dC(v) = [v final]·(C(v) - pcom(v)),
//   delta(u, a) = (dC(v) + U(v)) - U(u) with v = δ(u, a) (full AC transition), all in fp32.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <string>
#include <vector>

#include "flexctc_internal.h"

namespace flexctc {

flexctc_status build_boost_host(const int32_t* toks, const int64_t* offs, int32_t n, float w, int32_t V,
                                BoostHost& out) {
    if (n <= 0) return fail(FLEXCTC_ERR_INVALID_ARG, "empty phrase list");
    if (!(w > 0.0f)) return fail(FLEXCTC_ERR_INVALID_ARG, "token_weight must be > 0");
    if (V < 1) return fail(FLEXCTC_ERR_INVALID_ARG, "vocab_size must be >= 1");
    if (!toks || !offs) return fail(FLEXCTC_ERR_INVALID_ARG, "null phrase arrays");
    // goto trie, children kept sorted by token
    std::vector<std::vector<std::pair<int32_t, int32_t>>> kids(1);
    std::vector<int32_t> depth{0}, parent{0};
    std::vector<uint8_t> final_{0};
    for (int32_t i = 0; i < n; ++i) {
        int64_t b = offs[i], e = offs[i + 1];
        if (e <= b) return fail(FLEXCTC_ERR_INVALID_ARG, "empty phrase " + std::to_string(i));
        int32_t u = 0;
        for (int64_t j = b; j < e; ++j) {
            int32_t a = toks[j];
            if (a < 0 || a >= V)
                return fail(FLEXCTC_ERR_INVALID_ARG, "phrase " + std::to_string(i) + " has a token outside [0, V) (blank is V)");
            auto& ks = kids[u];
            auto it = std::lower_bound(ks.begin(), ks.end(), std::make_pair(a, INT32_MIN));
            if (it != ks.end() && it->first == a) {
                u = it->second;
            } else {
                int32_t v = (int32_t)kids.size();
                ks.insert(it, {a, v});
                kids.emplace_back();
                depth.push_back(depth[u] + 1);
                parent.push_back(u);
                final_.push_back(0);
                u = v;
            }
        }
        final_[u] = 1;
    }
    const int32_t N = (int32_t)kids.size();
    if ((int64_t)N * V > (int64_t)INT32_MAX) return fail(FLEXCTC_ERR_CAPACITY, "boost table nodes*V > 2^31");
    // BFS order, failure links and the full transition table δ (goto, else δ(fail(u), a))
    std::vector<int32_t> bfs;
    bfs.reserve(N);
    bfs.push_back(0);
    for (size_t q = 0; q < bfs.size(); ++q)
        for (auto& kv : kids[bfs[q]]) bfs.push_back(kv.second);
    std::vector<int32_t> fail_(N, 0), nxt((size_t)N * V, 0);
    for (int32_t u : bfs) {
        int32_t* row = &nxt[(size_t)u * V];
        if (u != 0) memcpy(row, &nxt[(size_t)fail_[u] * V], sizeof(int32_t) * V);
        for (auto& kv : kids[u]) {
            if (u != 0) fail_[kv.second] = nxt[(size_t)fail_[u] * V + kv.first];
            row[kv.first] = kv.second;
        }
    }
    // reward law (R17) in fp32
    std::vector<float> C(N), committed(N), pcom(N), U(N), dC(N), gain(N);
    for (int32_t u : bfs) {
        C[u] = w * (float)depth[u];
        if (u == 0) { committed[u] = 0.0f; pcom[u] = 0.0f; }
        else {
            pcom[u] = committed[parent[u]];
            committed[u] = final_[u] ? C[u] : committed[parent[u]];
        }
        U[u] = C[u] - committed[u];
        dC[u] = final_[u] ? C[u] - pcom[u] : 0.0f;
        gain[u] = dC[u] + U[u];
    }
    out = BoostHost();
    out.V = V;
    out.N = N;
    out.tab.resize((size_t)N * V * 2);
    out.U = U;
    out.maxd.resize(N);
    for (int32_t u = 0; u < N; ++u) {
        float m = -INFINITY;
        for (int32_t a = 0; a < V; ++a) {
            int32_t v = nxt[(size_t)u * V + a];
            float d = gain[v] - U[u];
            out.tab[((size_t)u * V + a) * 2] = v;
            memcpy(&out.tab[((size_t)u * V + a) * 2 + 1], &d, 4);
            m = std::max(m, d);
        }
        out.maxd[u] = m;
    }
    // exception signature: bit lm_sig_bit(a) set for every token a whose transition from u differs
    // from the root's. For any other token, δ(u, a) = δ(root, a) and
    // delta(u, a) = fl(gain(δ(root, a)) - U(u)) = fl(delta(root, a) - U(u)) exactly (delta(root, a) =
    // gain(δ(root, a)) since U(root) = 0), so the device needs only the root row and U(u).
    out.sig.assign(N, 0ull);
    for (int32_t u = 1; u < N; ++u)
        for (int32_t a = 0; a < V; ++a)
            if (nxt[(size_t)u * V + a] != nxt[a]) out.sig[u] |= 1ull << lm_sig_bit(a);
    return FLEXCTC_OK;
}

}  // namespace flexctc
