// Merge-before-TopK variant of the frame step (config merge_first = 1; reading R27,
// SURVEY §8(f) NEXT 2): BJ north_star "merges duplicate prefixes by prefix hash, selects the
// top-K of the K×(V+1) candidates", against Alg. 1's TopK -> recombine order.
//
// Per frame t < L_b, one CTA per utterance:
//   every candidate (slot k, token w) of Eq. (1) (reading R19 order) joins the
//   group of its (transcript', last label) (R12 key); a group's score is the R13/R14 combiner
//   over its members ordered by (score desc, flat index asc); the K best groups by (merged score
//   desc, flat index of the best member asc) survive, then the θ-prune against fl(best - θ)
//   (P:138-139); the best member is the survivor (backpointer, label, LM/BT state).
//
// The groups have a fixed structure (no hash table is needed). With distinct (hash, last) slots,
// a transcript q has at most two live slots, (q, ∅) and (q, end(q)) — a "class". Groups:
//   * blank group of class P: the blank extensions of P's slots (<= 2 members);
//   * repeat group of slot k = (q, c), c != ∅: its repeat, plus the emissions of c from the slots
//     of the class whose transcript is q minus its last token (partners: hash_extend(h_j, c) ==
//     h_k, last_j != c) — exact for every such k, always evaluated (<= K groups);
//   * emission group (P, c) that no slot's repeat group owns: the emissions of c from P's slots
//     with last != c (1 or 2 members, sharing the LM / BT terms of P's state).
// Exact pre-prune of the emission groups: the special groups (blank, repeat) are scored exactly
// first; τ = max(fl(best - θ), K-th best special score) lower-bounds the final cut. An emission
// group can reach at most max_acc(P) + D[c] + β + α_LM·ub(P) + α_BT·maxd(P) (+ ln 2 for two
// members under log-sum-exp) + a rounding margin; below τ it can neither enter the top K nor
// survive the prune, and its members belong to no other group, so it is skipped. Everything
// above is scored exactly into a shared-memory buffer of (key, payload) entries; a full buffer is
// sorted and cut to its K best (the cut raises τ), so any number of groups fits.
// Not a throughput path: the variant exists for parity with the oracle's merge_first flag; the
// frame row is read with plain coalesced loads and the backtrace walks the pointers serially.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "device_common.cuh"
#include "flexctc_internal.h"

namespace flexctc {
namespace {

using namespace dev;

constexpr int kNT = 256;     // threads per CTA
constexpr int kCap = 2048;   // group buffer entries (power of two: bitonic sort)
constexpr int kSlab = kNT * 2;  // emission pairs examined per round (<= pushes per round)

struct MfPay { int slot, label, lmn, btn; };  // survivor member and the states after the frame

// bitonic sort of keys[0..n) descending (n a power of two), payload indices along
__device__ void sort_desc(uint64_t* keys, int* idx, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const bool desc = (i & k) == 0;
                    const uint64_t a = keys[i], b = keys[l];
                    if (desc ? a < b : a > b) {
                        keys[i] = b; keys[l] = a;
                        const int t = idx[i]; idx[i] = idx[l]; idx[l] = t;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ float lse_combine(float* s, int n, int merge_mode) {  // s sorted desc (R14)
    const float s0 = s[0];
    if (merge_mode == 1 || n == 1) return s0;
    float sum = 0.0f;
    for (int i = 1; i < n; ++i) sum = __fadd_rn(sum, (float)exp((double)__fsub_rn(s[i], s0)));
    return __fadd_rn(s0, (float)log1p((double)sum));
}

// members (score, flat) -> ordered by (score desc, flat asc); returns the group score, rep = index
__device__ __forceinline__ float group_of(float* s, uint32_t* f, int n, int merge_mode, int& rep) {
    for (int i = 1; i < n; ++i)  // insertion sort of <= 3 members
        for (int j = i; j > 0 && (s[j] > s[j - 1] || (s[j] == s[j - 1] && f[j] < f[j - 1])); --j) {
            const float ts = s[j]; s[j] = s[j - 1]; s[j - 1] = ts;
            const uint32_t tf = f[j]; f[j] = f[j - 1]; f[j - 1] = tf;
        }
    rep = 0;
    return lse_combine(s, n, merge_mode);
}

template <int LMV>
__global__ void __launch_bounds__(kNT) merge_first_kernel(const DecodeParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint64_t s_key[kCap];
    __shared__ int s_idx[kCap];
    __shared__ int s_cnt, s_nsel, s_best_slot;
    __shared__ float s_tau;
    __shared__ float s_red[kNT / 32];
    __shared__ int s_creps[kMaxBeam], s_corder[kMaxBeam], s_m1[kMaxBeam], s_ncls;
    __shared__ float s_cub[kMaxBeam];
    __shared__ uint64_t s_wkey[kNT / 32];
    __shared__ int s_wstar;
    const int tid = threadIdx.x;
    const int K = p.K, Vp1 = p.Vp1, blank = Vp1 - 1, V = Vp1 - 1;
    const bool lm_on = p.use_lm != 0, bt_on = p.use_bt != 0;
    const int b = p.order[blockIdx.x];
    const int L = p.len_c[b];
    const int64_t bp_base = (int64_t)b * p.T * K;
    const int RW4 = lm_on ? p.lm.RW / 4 : 0;

    // shared layout: row, two banks of slot state, per-slot scratch, payloads
    unsigned char* q = smem_raw;
    auto take = [&](size_t bytes) { unsigned char* r = q; q += (bytes + 15) & ~size_t(15); return r; };
    float* row = (float*)take(4 * (size_t)Vp1);
    float* acc = (float*)take(8 * K);        // [2][K]
    int* last = (int*)take(8 * K);
    uint64_t* hsh = (uint64_t*)take(16 * K);
    int* lms = (int*)take(8 * K);
    int* bts = (int*)take(8 * K);
    int* cls = (int*)take(4 * K);            // class representative (lowest live slot with the same hash)
    int* own = (int*)take(4 * K);            // repeat group of slot k owns emission (own[k], last[k]) (-1: none)
    float* fsc = (float*)take(4 * K);        // final scores (EOS)
    MfPay* pay = (MfPay*)take(sizeof(MfPay) * kCap);

    int cb = 0;  // current bank
    int rdy = 0;  // streamed input: frames this thread has seen landed
    for (int k = tid; k < K; k += kNT) {
        acc[k] = k == 0 ? 0.0f : kNeg;
        last[k] = blank;                 // R6
        hsh[k] = 0ull;
        lms[k] = lm_on ? p.lm.start : 0;
        bts[k] = 0;
    }
    __syncthreads();

    auto recp = [&](int state) -> const int* { return (const int*)(p.lm.rec + (size_t)state * RW4); };
    // LM / BT terms of token w from states (ls, bs): {lm logp, next}, {bt delta, next}
    auto fusion = [&](int ls, int bs, int w, float& lp, int& ln, float& bd, int& bn) {
        lp = 0.0f; ln = ls; bd = 0.0f; bn = bs;
        if (bt_on) { const int2 e = __ldg(&p.bt.tab[(size_t)bs * V + w]); bn = e.x; bd = __int_as_float(e.y); }
        if (lm_on) lp = lm_query<LMV>(p.lm, recp(ls), w, ln);
    };
    // Eq. (1) emission score (R19 order)
    auto emit_score = [&](float a, float d, float lp, float bd) -> float {
        float s = __fadd_rn(__fadd_rn(a, d), p.beta);
        if (lm_on) s = __fmaf_rn(p.alpha_lm, lp, s);
        if (bt_on) s = __fmaf_rn(p.alpha_bt, bd, s);
        return s;
    };
    auto push = [&](float score, uint32_t flat, MfPay py) {
        const int j = atomicAdd(&s_cnt, 1);
        s_key[j] = make_key(score, flat);
        s_idx[j] = j;
        pay[j] = py;
    };
    // keep the K best buffer entries (sorted, compacted to the front); returns the K-th score or -inf
    auto cut_to_k = [&]() {
        __syncthreads();
        const int n = s_cnt;
        if (n <= kNT) {
            // rank selection (the keys are distinct: each group's best member is its own): one
            // entry per thread, its rank among the n by one pass over the keys, the K best written
            // to their ranks — two barriers instead of the sorting network's log^2 n / 2
            uint64_t kk = 0ull;
            MfPay pp{};
            int r = kNT;
            if (tid < n) {
                kk = s_key[tid];
                pp = pay[tid];
                r = 0;
                for (int j = 0; j < n; ++j) r += s_key[j] > kk ? 1 : 0;
            }
            __syncthreads();
            if (r < K) { s_key[r] = kk; s_idx[r] = r; pay[r] = pp; }
            __syncthreads();
            if (tid == 0) {
                const int keep = min(n, K);
                s_cnt = keep;
                if (keep == K) s_tau = fmaxf(s_tau, score_of(s_key[K - 1]));
            }
            __syncthreads();
            return;
        }
        int n2 = 2;
        while (n2 < n) n2 <<= 1;
        for (int i = n + tid; i < n2; i += kNT) { s_key[i] = 0ull; s_idx[i] = i; }
        __syncthreads();
        sort_desc(s_key, s_idx, n2);
        // move the payloads of the K best to the front (via registers: K <= kNT)
        MfPay mine{};
        const int keep = min(n, K);
        if (tid < keep) mine = pay[s_idx[tid]];
        __syncthreads();
        if (tid < keep) { pay[tid] = mine; s_idx[tid] = tid; }
        if (tid == 0) {
            s_cnt = keep;
            if (keep == K) s_tau = fmaxf(s_tau, score_of(s_key[K - 1]));
        }
        __syncthreads();
    };

    for (int t = 0; t < L; ++t) {
        const int nb = cb ^ 1;
        float* ca = acc + cb * K; int* cl = last + cb * K; uint64_t* ch = hsh + cb * K;
        int* cls_l = lms + cb * K; int* cbs = bts + cb * K;
        const float* Dt = p.log_probs + (int64_t)b * p.stride_b + (int64_t)t * p.stride_t;
        wait_ready(p, blockIdx.x, t, rdy);  // streamed host input (flexctc_decode_host)
        for (int w = tid; w < Vp1; w += kNT) row[w] = p.ready ? Dt[w] : __ldg(&Dt[w]);  // P:126 D[:, t, :]
        if (tid == 0) { s_cnt = 0; s_tau = kNeg; }
        // ---- slot structure: classes, owners, class maxima
        for (int k = tid; k < K; k += kNT) {
            int c = -1, o = -1;
            if (ca[k] > kNeg) {
                for (int j = 0; j < K && c < 0; ++j)
                    if (ca[j] > kNeg && ch[j] == ch[k]) c = j;
                const int lk = cl[k];
                if (lk != blank)
                    for (int j = 0; j < K && o < 0; ++j)
                        if (ca[j] > kNeg && cl[j] != lk && hash_extend(ch[j], lk) == ch[k]) o = j;
            }
            cls[k] = c;
            own[k] = o;
        }
        __syncthreads();
        for (int k = tid; k < K; k += kNT)
            if (own[k] >= 0) own[k] = cls[own[k]];  // the partners' class
        __syncthreads();
        // ---- special groups, exactly: blank group per class, repeat group per slot with last != ∅
        for (int k = tid; k < K; k += kNT) {
            if (ca[k] == kNeg) continue;
            if (cls[k] == k) {  // blank group of class k
                float s[2]; uint32_t f[2]; int n = 0;
                for (int j = k; j < K && n < 2; ++j)
                    if (cls[j] == k) { s[n] = __fadd_rn(ca[j], row[blank]); f[n] = (uint32_t)j * Vp1 + blank; ++n; }
                int r;
                const float g = group_of(s, f, n, p.merge_mode, r);
                const int rs = (int)(f[r] / Vp1);
                push(g, f[r], MfPay{rs, blank, cls_l[rs], cbs[rs]});
            }
            const int c = cl[k];
            if (c != blank) {  // repeat group of slot k
                float s[3]; uint32_t f[3]; int n = 0;
                float rp = __fadd_rn(ca[k], row[c]);
                if (p.fuse_rep) {  // P:167 variant: LM / BT on the repeated emission (no β, no advance)
                    float lp, bd; int ln, bn;
                    fusion(cls_l[k], cbs[k], c, lp, ln, bd, bn);
                    if (lm_on) rp = __fmaf_rn(p.alpha_lm, lp, rp);
                    if (bt_on) rp = __fmaf_rn(p.alpha_bt, bd, rp);
                }
                s[n] = rp; f[n] = (uint32_t)k * Vp1 + c; ++n;
                const int P = own[k];
                if (P >= 0) {
                    float lp, bd; int ln, bn;
                    fusion(cls_l[P], cbs[P], c, lp, ln, bd, bn);  // shared by P's members
                    for (int j = P; j < K && n < 3; ++j)
                        if (cls[j] == P && cl[j] != c) {
                            s[n] = emit_score(ca[j], row[c], lp, bd);
                            f[n] = (uint32_t)j * Vp1 + c;
                            ++n;
                        }
                }
                int r;
                const float g = group_of(s, f, n, p.merge_mode, r);
                push(g, f[r], MfPay{(int)(f[r] / Vp1), c, cls_l[k], cbs[k]});  // states of q (= k's)
            }
        }
        __syncthreads();
        // τ0 = max(fl(best - θ), K-th best special group)
        {
            float m = kNeg;
            for (int i = tid; i < s_cnt; i += kNT) m = fmaxf(m, score_of(s_key[i]));
#pragma unroll
            for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if ((tid & 31) == 0) s_red[tid >> 5] = m;
            __syncthreads();
            if (tid == 0) {
                float mm = s_red[0];
                for (int i = 1; i < kNT / 32; ++i) mm = fmaxf(mm, s_red[i]);
                if (mm > kNeg) s_tau = fmaxf(s_tau, __fsub_rn(mm, p.theta));
            }
            __syncthreads();
            if (s_cnt >= K) cut_to_k();  // raises τ to the K-th special score
        }
        // ---- emission groups (P, c) no repeat group owns, pre-pruned by their bound
        // per live class (representative P): its <= 2 members and the token-independent part of
        // the bound, max acc + β + α_LM·ub(P) + α_BT·maxd(P) (+ ln 2 with two lse members)
        const bool no_bound = (lm_on && p.alpha_lm < 0.0f) || (bt_on && p.alpha_bt < 0.0f);
        if (tid == 0) {
            int nc = 0;
            for (int k = 0; k < K; ++k)
                if (cls[k] == k) s_creps[nc++] = k;
            s_ncls = nc;
        }
        for (int k = tid; k < K; k += kNT) {
            if (cls[k] != k) continue;
            int m0 = k, m1 = -1;
            for (int j = k + 1; j < K && m1 < 0; ++j)
                if (cls[j] == k) m1 = j;
            float ub = __fadd_rn(fmaxf(ca[m0], m1 >= 0 ? ca[m1] : kNeg), p.beta);
            if (lm_on) ub = __fadd_rn(ub, p.alpha_lm * __int_as_float(recp(cls_l[k])[4]));
            if (bt_on) ub = __fadd_rn(ub, p.alpha_bt * __ldg(&p.bt.maxd[cbs[k]]));
            if (m1 >= 0 && p.merge_mode == 0) ub = __fadd_rn(ub, 0.6931472f);
            s_cub[k] = ub;
            s_m1[k] = m1;
        }
        __syncthreads();
        const int ncls = s_ncls;
        // best-token stage (raises τ before the bulk filter, as the TopK-first kernels' stage A):
        // the frame's best non-blank token w* scored exactly for every live class in one round of
        // lookups; these groups are excluded from the bulk pass below
        {
            float bv = kNeg;
            int bw = -1;
            for (int w = tid; w < V; w += kNT)
                if (row[w] > bv || (row[w] == bv && bw >= 0 && w < bw)) { bv = row[w]; bw = w; }
            uint64_t key = bw >= 0 ? make_key(bv, (uint32_t)bw) : 0ull;
#pragma unroll
            for (int o = 16; o; o >>= 1) key = umax64(key, __shfl_xor_sync(0xffffffffu, key, o));
            if ((tid & 31) == 0) s_wkey[tid >> 5] = key;
            __syncthreads();
            if (tid == 0) {
                uint64_t k2 = s_wkey[0];
                for (int i = 1; i < kNT / 32; ++i) k2 = umax64(k2, s_wkey[i]);
                s_wstar = k2 ? (int)flat_of(k2) : -1;
            }
            __syncthreads();
        }
        const int wstar = s_wstar;
        auto emission_group = [&](int P, int c, float tau) {
            // members: P's slots whose last label is not c (a slot with last == c repeats)
            int mem[2]; int n = 0;
            if (cl[P] != c) mem[n++] = P;
            const int m1 = s_m1[P];
            if (m1 >= 0 && cl[m1] != c) mem[n++] = m1;
            if (n == 0) return;
            bool owned = false;
            for (int k = 0; k < K && !owned; ++k) owned = own[k] == P && cl[k] == c && ca[k] > kNeg;
            if (owned) return;
            float lp, bd; int ln, bn;
            fusion(cls_l[P], cbs[P], c, lp, ln, bd, bn);
            float s[2]; uint32_t f[2];
            for (int m = 0; m < n; ++m) { s[m] = emit_score(ca[mem[m]], row[c], lp, bd); f[m] = (uint32_t)mem[m] * Vp1 + c; }
            int r;
            const float g = group_of(s, f, n, p.merge_mode, r);
            if (g == kNeg || g < tau) return;  // below a lower bound of the final cut
            push(g, f[r], MfPay{(int)(f[r] / Vp1), c, ln, bn});
        };
        if (wstar >= 0) {
            for (int ci = tid; ci < ncls; ci += kNT) emission_group(s_creps[ci], wstar, s_tau);
            __syncthreads();
            if (s_cnt >= K) cut_to_k();
        }
        // bulk pass: classes in order of their bound (cub desc); a class whose bound with the
        // frame's best token cannot reach τ ends the pass (every later class is weaker), and τ is
        // raised to the K-th best group after every class (threshold algorithm)
        for (int ci = tid; ci < ncls; ci += kNT) {
            const int P = s_creps[ci];
            const float u = s_cub[P];
            int r = 0;
            for (int cj = 0; cj < ncls; ++cj) {
                const float v = s_cub[s_creps[cj]];
                r += (v > u || (v == u && cj < ci)) ? 1 : 0;
            }
            s_corder[r] = P;
        }
        __syncthreads();
        const float dmax = wstar >= 0 ? row[wstar] : kNeg;
        for (int ci = 0; ci < ncls; ++ci) {
            const int P = s_corder[ci];
            if (!no_bound && s_tau > kNeg) {
                float ub = __fadd_rn(s_cub[P], dmax);
                ub += 1e-3f + 1e-5f * fabsf(ub);
                if (ub < s_tau) break;  // uniform: s_tau was last written before a barrier
            }
            for (int c0 = 0; c0 < V; c0 += kSlab) {
                if (s_cnt + kSlab > kCap) cut_to_k();
                const float tau = s_tau;
                for (int c = c0 + tid; c < min(V, c0 + kSlab); c += kNT) {
                    if (c == wstar) continue;  // scored in the best-token stage
                    if (!no_bound && tau > kNeg) {
                        float ub = __fadd_rn(s_cub[P], row[c]);
                        ub += 1e-3f + 1e-5f * fabsf(ub);  // rounding margin
                        if (ub < tau) continue;
                    }
                    emission_group(P, c, tau);
                }
                __syncthreads();
            }
            if (s_cnt > K) cut_to_k();
        }
        // ---- TopK over the groups, θ-prune, beams.update
        cut_to_k();
        const int nsel = s_cnt;
        const float best = nsel > 0 ? score_of(s_key[0]) : kNeg;
        const float thr = __fsub_rn(best, p.theta);  // R10
        float* na = acc + nb * K; int* nl = last + nb * K; uint64_t* nh = hsh + nb * K;
        int* nlm = lms + nb * K; int* nbt = bts + nb * K;
        for (int i = tid; i < K; i += kNT) {
            uint8_t par = 0;
            uint16_t lab = (uint16_t)blank;
            if (i < nsel && score_of(s_key[i]) >= thr) {
                const MfPay py = pay[i];
                const int k = py.slot, w = py.label;
                na[i] = score_of(s_key[i]);
                nl[i] = w;
                nh[i] = (w != blank && w != cl[k]) ? hash_extend(ch[k], w) : ch[k];  // P:88, R5
                nlm[i] = py.lmn;
                nbt[i] = py.btn;
                par = (uint8_t)k;
                lab = (uint16_t)w;
            } else {
                na[i] = kNeg; nl[i] = blank; nh[i] = 0ull; nlm[i] = lm_on ? p.lm.start : 0; nbt[i] = 0;
            }
            p.bp_parent[bp_base + (int64_t)t * K + i] = par;
            p.bp_label[bp_base + (int64_t)t * K + i] = lab;
        }
        __syncthreads();
        cb = nb;
    }

    // ---- EOS, final merge by transcript across last labels (R15), 1-best
    float* ca = acc + cb * K; uint64_t* ch = hsh + cb * K;
    for (int k = tid; k < K; k += kNT) {
        float fs = ca[k];
        if (fs > kNeg) {
            if (lm_on) fs = __fmaf_rn(p.alpha_lm, __int_as_float(recp(lms[cb * K + k])[5]), fs);
            if (bt_on && p.retract) fs = __fmaf_rn(-p.alpha_bt, __ldg(&p.bt.U[bts[cb * K + k]]), fs);
        }
        fsc[k] = fs;
    }
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    for (int i = tid; i < K; i += kNT) {
        const float si = fsc[i];
        if (!(si > kNeg)) continue;
        bool dead = false;
        for (int j = 0; j < K && !dead; ++j)
            dead = j != i && fsc[j] > kNeg && ch[j] == ch[i] && (fsc[j] > si || (fsc[j] == si && j < i));
        if (dead) continue;
        float g = si;
        if (p.merge_mode == 0) {  // the other members in (score desc, slot asc) order: at most one
            float sum = 0.0f;
            bool any = false;
            for (int j = 0; j < K; ++j)
                if (j != i && fsc[j] > kNeg && ch[j] == ch[i]) { sum = __fadd_rn(sum, (float)exp((double)__fsub_rn(fsc[j], si))); any = true; }
            if (any) g = __fadd_rn(si, (float)log1p((double)sum));
        }
        const int j = atomicAdd(&s_cnt, 1);
        s_key[j] = make_key(g, (uint32_t)i);
    }
    __syncthreads();
    if (tid == 0) {
        uint64_t bk = 0ull;
        for (int j = 0; j < s_cnt; ++j) bk = umax64(bk, s_key[j]);
        s_best_slot = s_cnt > 0 ? (int)flat_of(bk) : -1;
        s_tau = s_cnt > 0 ? score_of(bk) : kNeg;
        s_nsel = 0;
        // backtrace: serial walk of the pointers
        int32_t* align = (p.out_align ? p.out_align : p.align_ws) + (int64_t)b * p.T;
        if (s_best_slot >= 0) {
            int s = s_best_slot;
            for (int t = L - 1; t >= 0; --t) {
                const int64_t o = bp_base + (int64_t)t * K + s;
                align[t] = p.bp_label[o];
                s = p.bp_parent[o];
            }
        }
        // collapse to tokens + timestamps (R20)
        int n = 0;
        int32_t* otok = p.out_tokens + (int64_t)b * p.T;
        int32_t* ots = p.out_ts ? p.out_ts + (int64_t)b * p.T : nullptr;
        if (s_best_slot >= 0)
            for (int t = 0; t < L; ++t) {
                const int at = align[t], ap = t ? align[t - 1] : blank;
                if (at != blank && at != ap) { otok[n] = at; if (ots) ots[n] = t; ++n; }
            }
        s_nsel = n;
        p.out_num[b] = n;
        p.out_scores[b] = s_tau;
    }
    __syncthreads();
    const int n = s_nsel;
    for (int i = n + tid; i < p.T; i += kNT) {
        p.out_tokens[(int64_t)b * p.T + i] = -1;
        if (p.out_ts) p.out_ts[(int64_t)b * p.T + i] = -1;
    }
    if (p.out_align)
        for (int i = (s_best_slot >= 0 ? L : 0) + tid; i < p.T; i += kNT) p.out_align[(int64_t)b * p.T + i] = -1;
}

}  // namespace

size_t merge_first_smem(int K, int Vp1) {
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    return al(4 * (size_t)Vp1) + al(8 * K) + al(8 * K) + al(16 * K) + al(8 * K) + al(8 * K) + al(4 * K) + al(4 * K) +
           al(4 * K) + al(sizeof(MfPay) * kCap);
}

// One CTA per utterance (blockIdx -> p.order, longest first); after order_kernel.
int launch_merge_first(const DecodeParams& p, void* stream, void* ev0, void* ev1, std::string& err) {
    if (p.B == 0) return 0;
    const size_t smem = merge_first_smem(p.K, p.Vp1);
    auto kern = p.use_lm && p.lm.NL > 2 ? merge_first_kernel<kMaxLmLevels> : merge_first_kernel<2>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    cudaStream_t st = (cudaStream_t)stream;
    if (ev0 && ev1) cudaEventRecord((cudaEvent_t)ev0, st);
    kern<<<p.B, kNT, smem, st>>>(p);
    set_kernel_name("merge_first_kernel");
    e = cudaGetLastError();
    if (e == cudaSuccess && ev0 && ev1) cudaEventRecord((cudaEvent_t)ev1, st);
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    return 0;
}

}  // namespace flexctc
