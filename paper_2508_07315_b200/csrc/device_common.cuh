// Device helpers shared by the beam kernel (beam_kernel.cu) and the greedy kernels
// (greedy_kernel.cu): orderable score keys, cp.async row staging, the NGPU-LM arc query.
// Product code only; nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "flexctc_internal.h"

namespace flexctc {
namespace dev {

constexpr float kNeg = -INFINITY;

__device__ __forceinline__ uint64_t hash_extend(uint64_t h, int w) {  // SPEC S:58 (FNV-64 prime)
    return (h ^ (uint64_t)(w + 1)) * 1099511628211ull;
}

__device__ __forceinline__ uint32_t ord_of(float s) {
    uint32_t u = __float_as_uint(s);
    if (u == 0x80000000u) u = 0u;  // -0 == +0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float score_of(uint64_t key) {
    const uint32_t o = (uint32_t)(key >> 32);
    const uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(u);
}
__device__ __forceinline__ uint64_t make_key(float s, uint32_t f) {
    return ((uint64_t)ord_of(s) << 32) | (uint64_t)(0xffffffffu - f);
}
__device__ __forceinline__ uint32_t flat_of(uint64_t key) { return 0xffffffffu - (uint32_t)key; }
// (slot k, token w) -> an index ordered exactly like the flat index k·V' + w (w < 2^16)
__device__ __forceinline__ uint32_t flat_idx(int k, int w) { return ((uint32_t)k << 16) | (uint32_t)w; }
__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

__device__ __forceinline__ void cp_async4(void* s, const void* g) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
// 16-B copy with an L2 evict-first policy (streamed data that must not displace L2-resident tables)
__device__ __forceinline__ void cp_async16_ef(void* s, const void* g, uint64_t pol) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "l"(pol));
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// NGPU-LM query from a cached state record: log P(w | state) and the next state.
// All arc levels (contexts of length >= 2) are binary-searched in lockstep (their loads are
// independent), the level-1 dense row is loaded in parallel, and the first level holding w
// wins; cum values are the fp32 backoff sums of the sequential walk (lm_query_host, R19).
template <int LMV>  // max arc levels (order - 2)
__device__ __forceinline__ float lm_query(const LmDev& lm, const int* __restrict__ rec, int w, int& next) {
    const int u = rec[1];
    int2 d = make_int2(0, 0);
    if (u >= 0) d = __ldg(&lm.dense[(size_t)u * lm.V + w]);
    // signature: no arc level holds w -> skip the searches (same result: the dense / root level)
    const uint32_t sw = (uint32_t)rec[6 + (lm_sig_bit(w) >> 5)];
    const int n = ((sw >> (lm_sig_bit(w) & 31)) & 1u) ? rec[0] : 0;
    int lo[LMV], hi[LMV], hlp[LMV], hnx[LMV];
    bool hit[LMV];
#pragma unroll
    for (int j = 0; j < LMV; ++j) {
        lo[j] = j < n ? rec[8 + 3 * j] : 0;
        hi[j] = j < n ? lo[j] + rec[8 + 3 * j + 1] : 0;
        hit[j] = false;
        hlp[j] = 0;
        hnx[j] = 0;
    }
    for (;;) {
        bool any = false;
#pragma unroll
        for (int j = 0; j < LMV; ++j) {
            if (lo[j] < hi[j]) {
                any = true;
                const int mid = (lo[j] + hi[j]) >> 1;
                const int4 a = __ldg(&lm.arcs[mid]);  // the whole arc: a hit needs no reload
                if (a.x == w) { hit[j] = true; hlp[j] = a.y; hnx[j] = a.z; hi[j] = lo[j]; }
                else if (a.x < w) lo[j] = mid + 1;
                else hi[j] = mid;
            }
        }
        if (!any) break;
    }
#pragma unroll
    for (int j = 0; j < LMV; ++j) {
        if (hit[j]) {
            next = hnx[j];
            return __fadd_rn(__int_as_float(rec[8 + 3 * j + 2]), __int_as_float(hlp[j]));
        }
    }
    if (u >= 0) {
        const bool found = (d.y & 0x80000000) != 0;
        next = d.y & 0x7fffffff;
        return __fadd_rn(__int_as_float(found ? rec[2] : rec[3]), __int_as_float(d.x));
    }
    next = __ldg(&lm.uni_next[w]);
    return __fadd_rn(__int_as_float(rec[3]), __ldg(&lm.uni_lp[w]));
}

// A ring slot holds one frame row at float offset row_off(src) (0..3) so that shared and global
// addresses agree mod 16 B: every row, aligned or not (4100-B rows at V' = 1025), is copied with
// 16-B cp.async except for <= 3 head and tail elements.
__device__ __forceinline__ int row_off(const float* src) { return (int)(((uintptr_t)src >> 2) & 3); }

// issued by `nt` threads with local index `tid` (all threads, or the helper warps)
// overread: the buffer is library-owned (16-B aligned, >= 16 B of slack after the last row), so
// the row is covered by whole 16-B blocks, the neighbouring rows' bytes landing unused in the slot.
__device__ __forceinline__ void load_row(float* slot, const float* src, int Vp1, int tid, int nt, int overread) {
    const int off = row_off(src);
    const uint64_t pol = policy_evict_first();  // D is read once: keep the LM / boost tables in L2
    if (overread) {
        const float* g = src - off;
        const int n16 = (off + Vp1 + 3) >> 2;
        for (int i = tid; i < n16; i += nt) cp_async16_ef(slot + 4 * i, g + 4 * i, pol);
        return;
    }
    float* dst = slot + off;
    const int h = min((4 - off) & 3, Vp1);
    if (tid < h) cp_async4(dst + tid, src + tid);
    const int n4 = (Vp1 - h) >> 2;
    for (int i = tid; i < n4; i += nt) cp_async16_ef(dst + h + 4 * i, src + h + 4 * i, pol);
    const int t0 = h + 4 * n4;
    if (t0 + tid < Vp1) cp_async4(dst + t0 + tid, src + t0 + tid);
}

// bf16 logits row into a 16-B aligned staging area: the row's covering 16-B blocks by cp.async
// (row element w at dst + (src mod 16) + 2w) when they lie inside [lo, hi), else (the tensor's
// first / last row) plain element copies, visible after the caller's barrier. Plain cp.async.cg:
// the same copy with an L2::cache_hint evict-first policy raised "illegal instruction" on the B200
// in this kernel (the fp32 rows' copies carry the hint without trouble), so the logits ride the
// default L2 policy.
__device__ __forceinline__ void load_row_bf16(char* dst, const uint16_t* src, int Vp1, int tid, int nt, const char* lo,
                                              const char* hi) {
    const char* s = (const char*)src;
    const char* g = (const char*)((uintptr_t)s & ~(uintptr_t)15);
    const int nb16 = (int)(((s - g) + 2 * Vp1 + 15) >> 4);
    if (g >= lo && g + 16 * (size_t)nb16 <= hi) {
        for (int i = tid; i < nb16; i += nt) cp_async16(dst + 16 * i, g + 16 * i);
    } else {
        for (int w = tid; w < Vp1; w += nt) *(uint16_t*)(dst + (s - g) + 2 * w) = __ldg(src + w);
    }
}

// Streamed input (flexctc_decode_host): wait until frame r of the utterance at LPT position u has
// landed. First wave (u < p.wave, or p.wave = 0): ready[0] > r (frames sent frame-major); later
// utterances: ready[1] > u - p.wave (sent whole, in LPT order). `ready` caches what this thread
// has seen for the current utterance (reset per utterance). A 10 s watchdog flags
// FLEXCTC_FLAG_STREAM_TIMEOUT instead of hanging the device.
__device__ __forceinline__ void wait_ready(const DecodeParams& p, int u, int r, int& ready) {
    if (!p.ready || r < ready) return;
    const bool whole = p.wave > 0 && u >= p.wave;
    const uint32_t* word = p.ready + (whole ? 1 : 0);
    const int need = whole ? u - p.wave : r;
    const long long t0 = clock64();
    uint32_t v;
    for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(word) : "memory");
        if ((int)v > need) { if (whole) v = 0x7fffffffu; break; }
        if (clock64() - t0 > 20000000000ll) {
            atomicOr(p.flags, FLEXCTC_FLAG_STREAM_TIMEOUT);
            v = 0x7fffffffu;
            break;
        }
        __nanosleep(200);
    }
    ready = (int)v;
}

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier ----------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// orders this thread's generic-proxy shared accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// the same with an L2 cache policy (createpolicy), e.g. evict-first for data read once
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    } while (!ok);
}

// One frame row into a 16-B aligned ring slot at float offset row_off(src) (the layout of
// load_row), called by all 32 lanes of a warp: lane 0 issues a single bulk copy of the row's
// covering 16-B blocks when those lie inside [lo, hi) (the tensor's bytes: nothing outside the
// caller's buffer is read); otherwise (at most the first and the last row of a tensor) the warp
// copies the row with plain loads and lane 0 arrives without a transaction count.
// Completion: mbarrier `bar` (count 1).
__device__ __forceinline__ void bulk_row(float* slot, const float* src, int Vp1, uint64_t* bar, const char* lo,
                                         const char* hi, int lane) {
    const int off = row_off(src);
    const char* g = (const char*)(src - off);
    const uint32_t bytes = (uint32_t)(((off + Vp1) * 4 + 15) & ~15);
    if (g >= lo && g + bytes <= hi) {
        if (lane == 0) {
            fence_proxy_async();  // earlier generic reads of this slot before the async write
            mbar_arrive_tx(bar, bytes);
            bulk_g2s(slot, g, bytes, bar);
        }
    } else {
        for (int w = lane; w < Vp1; w += 32) slot[off + w] = __ldg(src + w);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
    }
}

// ---- bf16 logits input (reading R25) ---------------------------------
__device__ __forceinline__ float bf16f(uint16_t x) { return __uint_as_float((uint32_t)x << 16); }

// per-CTA device counters (SURVEY §5 "device counters"), flushed per utterance
enum Stat { kFrames, kAlive, kListed, kEvalSparse, kDenseFrames, kRowsBuilt, kEvalDense, kCompactions,
            kStageA, kDeferredNext,
            // SM cycles (thread 0) per frame phase: 1-3, 4, LM row builds (inside 4), 5, 6-7;
            // frames with listed tokens and their cycles
            kCycP13, kCycP4, kCycRows, kCycP5, kCycP67, kHeavyFrames, kCycHeavy,
            // finer split: frame top (row issue + wait), phase 2, phase 3, phase 4 setup / collect / evaluate
            kCycTop, kCycP2, kCycP3, kCycP4Setup, kCycP4Collect, kCycP4Eval,
            // frames without listed tokens: count and cycles of phase 1, 2, 3, B1 (+ phase-4 entry),
            // 5, 6, 7
            kLightFrames, kLP1, kLP2, kLP3, kLB1, kLP5, kLP6, kLP7,
            // phase 7 of those frames: match.any, merge scores, chunk ancestors + records, final sync
            kLP7a, kLP7b, kLP7c, kLP7d,
            // frames taken by the CTA kernel's settled-beam fast path
            kFastFrames, kCycFast, kNumStats };

}  // namespace dev
}  // namespace flexctc
