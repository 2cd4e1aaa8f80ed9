"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element, on seeded
synthetic inputs shaped like the paper's workloads, plus edge cases and
size-independent invariants. Tokens, timestamps and alignments must be identical; scores within
1e-4 absolute (BASELINE.json north_star), bit-identical in max mode."""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2508_07315_b200 as F  # noqa: E402
import synth  # noqa: E402
from tests.conftest import GOLDEN  # noqa: E402
from tests.exact.ctc_exact import greedy  # noqa: E402

TOL = 1e-4
NTH = os.cpu_count() or 4


def gpu_decode(D, L, cfg, lm=None, bt=None, Vp1=None, alignment=True):
    Dt = torch.from_numpy(np.ascontiguousarray(D)).cuda() if isinstance(D, np.ndarray) else D
    Lt = torch.from_numpy(np.asarray(L, dtype=np.int32)).cuda()
    out = F.decode(Dt, Lt, cfg, lm, bt, Vp1=Vp1, alignment=alignment)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def ocfg(c):
    return oracle.make_cfg(c.beam, c.alpha_lm, c.alpha_bt, c.beta, c.theta, c.merge_mode, c.retract_boost_at_eos,
                           c.fuse_repeats, c.merge_first)


def compare(g, o, idx=None, tol=TOL, bitwise=False, ctx=""):
    idx = range(len(o["num_tokens"])) if idx is None else idx
    worst = 0.0
    for j, b in enumerate(idx):
        n = int(o["num_tokens"][j])
        assert int(g["num_tokens"][b]) == n, (ctx, b)
        assert np.array_equal(g["tokens"][b], o["tokens"][j]), (ctx, b)
        assert np.array_equal(g["timestamps"][b], o["timestamps"][j]), (ctx, b)
        if "alignment" in o and "alignment" in g:
            assert np.array_equal(g["alignment"][b], o["alignment"][j]), (ctx, b)
        gs, os_ = float(g["scores"][b]), float(o["scores"][j])
        if math.isinf(os_):
            assert gs == os_
            continue
        worst = max(worst, abs(gs - os_))
        if bitwise:
            assert np.float32(gs) == np.float32(os_), (ctx, b, gs, os_)
        assert abs(gs - os_) <= tol, (ctx, b, gs, os_)
    return worst


def run_pair(D, L, cfg, glm=None, olm=None, gbt=None, obt=None, idx=None, Vp1=None, bitwise=None, ctx=""):
    g = gpu_decode(D, L, cfg, glm, gbt, Vp1=Vp1)
    Dn = D if Vp1 is None else D
    sub = np.asarray(list(idx)) if idx is not None else None
    Do = Dn if sub is None else Dn[sub]
    Lo = np.asarray(L) if sub is None else np.asarray(L)[sub]
    o = oracle.decode_strided(np.ascontiguousarray(Do), Vp1 or D.shape[2], Lo, ocfg(cfg), olm, obt, NTH,
                              with_alignment=True)
    if bitwise is None:
        bitwise = cfg.merge_mode == 1
    return compare(g, o, idx=sub, bitwise=bitwise, ctx=ctx), g, o


def wl_cfg(wl, **over):
    kw = dict(beam=wl.beam, alpha_lm=wl.alpha_lm if wl.lm else 0.0, alpha_bt=wl.alpha_bt if wl.boost else 0.0,
              beta=wl.beta, theta=wl.theta, merge_mode=wl.merge_mode)
    kw.update(over)
    return F.config(**kw)


# ------------------------------------------------------------------------ workload configs

@pytest.mark.parametrize("mode", [0, 1])
def test_c1_full(mode):
    wl, D, L, _, _ = synth.workload_inputs("c1")
    run_pair(D, L, wl_cfg(wl, merge_mode=mode), ctx="c1")


@pytest.mark.parametrize("mode", [0, 1])
def test_c2_full(mode):
    wl, D, L, _, _ = synth.workload_inputs("c2")
    run_pair(D, L, wl_cfg(wl, merge_mode=mode), ctx="c2")


def test_c2_beam_vs_greedy():
    """c2 also pins K=1 on the GPU against greedy decoding (PAPER Table II 'greedy' rows)."""
    wl, D, L, _, _ = synth.workload_inputs("c2")
    g = gpu_decode(D, L, F.config(1, theta=float("inf")))
    for b in range(wl.B):
        toks, score, _ = greedy(D[b, :L[b], :wl.Vp1], wl.V)
        assert tuple(g["tokens"][b, :g["num_tokens"][b]]) == toks
        assert np.float32(g["scores"][b]) == np.float32(score)


def test_fused_greedy_c4(lm_pair, bt_pair):
    """K = 1 with LM + boosting: the fused greedy decoder of PAPER Table II ('greedy' + LM/PB)."""
    wl, D, L, _, _ = synth.workload_inputs("c4")
    for mode in (0, 1):
        run_pair(D, L, wl_cfg(wl, beam=1, merge_mode=mode), lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1],
                 ctx=f"greedy-fused m{mode}")


def test_c3_full(lm_pair):
    wl, D, L, _, _ = synth.workload_inputs("c3")
    run_pair(D, L, wl_cfg(wl), glm=lm_pair[0], olm=lm_pair[1], ctx="c3")


@pytest.mark.parametrize("mode", [0, 1])
def test_c4_full(lm_pair, bt_pair, mode):
    """The bench workload (beam 16, 4-gram LM, 1000 phrases) at full size, every utterance."""
    wl, D, L, _, _ = synth.workload_inputs("c4")
    run_pair(D, L, wl_cfg(wl, merge_mode=mode), lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1], ctx="c4")


def test_c5_sampled(lm_pair, bt_pair):
    """B=512 LibriSpeech-shaped, K=128, LM + boosting: the GPU decodes the whole batch in one
    launch; the oracle checks a sample (the longest, the shortest and random utterances)."""
    wl, D, L, _, _ = synth.workload_inputs("c5")
    order = np.argsort(-L, kind="stable")
    rng = np.random.default_rng(0)
    idx = sorted(set([int(order[0]), int(order[-1])] + list(map(int, rng.choice(wl.B, 4, replace=False)))))
    run_pair(D, L, wl_cfg(wl), lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1], idx=idx, ctx="c5")


@pytest.mark.parametrize("nt,dense,solo", [("32", "1", None), ("32", None, None), ("64", "24", None),
                                           ("128", None, None), ("256", "1", None), ("256", None, "0"),
                                           ("256", "24", "0")])
def test_kernel_variants_c4(lm_pair, bt_pair, nt, dense, solo, monkeypatch):
    """Every launch variant (threads per utterance, LM row-cache dense path, beam-warp + helpers
    mode on/off) matches the oracle on c4 utterances (FLEXCTC_NT / FLEXCTC_DENSE_MIN /
    FLEXCTC_SOLO are tuning overrides)."""
    monkeypatch.setenv("FLEXCTC_WARP", "0")  # the persistent CTA kernel (K <= 32 defaults to the warp path)
    monkeypatch.setenv("FLEXCTC_NT", nt)
    if dense:
        monkeypatch.setenv("FLEXCTC_DENSE_MIN", dense)
    if solo:
        monkeypatch.setenv("FLEXCTC_SOLO", solo)
    wl, D, L, _, _ = synth.workload_inputs("c4", B=12)
    run_pair(D, L, wl_cfg(wl), lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1], ctx=f"nt{nt} dense{dense}")


# ------------------------------------------------------------------------ edge cases

def _small(rng, B, T, Vp1, peak=6.0, pad=0.0, stride=None):
    D = synth.random_logprobs(rng, B, T, Vp1, peak=peak).astype(np.float32)
    if stride is not None and stride > Vp1:
        E = np.full((B, T, stride), pad, np.float32)
        E[:, :, :Vp1] = D
        D = E
    return D


@pytest.mark.parametrize("K", [1, 2, 3, 7, 32, 33, 64, 100, 128, 256])
def test_beam_sizes_small_vocab(K):
    rng = np.random.default_rng(K)
    B, T, Vp1 = 6, 37, 11
    D = _small(rng, B, T, Vp1)
    L = np.array([37, 1, 0, 20, 36, 5])
    for mode in (0, 1):
        for theta in (12.0, 3.0, float("inf")):
            run_pair(D, L, F.config(K, beta=0.25, theta=theta, merge_mode=mode), ctx=f"K{K} th{theta} m{mode}")


def test_theta_inf_dense_path_with_lm_fixture():
    """θ = ∞ forces the dense path (every candidate scored, buffer compaction) with LM + BT."""
    syms = ["a", "b", "c"]
    p = os.path.join(GOLDEN, "arpa_3gram.arpa")
    glm, olm = F.LM(p, 3, syms, device=0), oracle.LM(p, 3, syms)
    phrases = [[0, 1], [1, 2], [0, 1, 2]]
    gbt, obt = F.Boost(phrases, 0.7, 3, device=0), oracle.Boost(phrases, 0.7, 3)
    rng = np.random.default_rng(3)
    D = _small(rng, 5, 30, 4, peak=2.0)
    L = np.array([30, 29, 1, 0, 17])
    for K in (1, 4, 16, 64, 256):
        for mode in (0, 1):
            for retract in (0, 1):
                cfg = F.config(K, alpha_lm=0.6, alpha_bt=0.8, beta=0.3, theta=float("inf"), merge_mode=mode,
                               retract_boost_at_eos=retract)
                run_pair(D, L, cfg, glm, olm, gbt, obt, ctx=f"K{K} m{mode} r{retract}")


def test_negative_weights_disable_preprune(lm_pair, bt_pair):
    wl, D, L, _, _ = synth.workload_inputs("c4", B=4)
    cfg = wl_cfg(wl, alpha_lm=-0.3, beta=-0.5)
    run_pair(D, L, cfg, lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1], ctx="neg")


def test_flat_stress_variant(lm_pair, bt_pair):
    """'flat' logits (target + U(4,8)): many tokens within θ, exercises buffer compaction."""
    wl = synth.WORKLOADS["c4"]
    L = np.array([120, 97, 64, 3], dtype=np.int32)
    D, _ = synth.logprobs(4, 120, wl.V, L, 77, synth.phrases(1024), flat=True)
    for K in (16, 128):
        run_pair(D, L, wl_cfg(wl, beam=K), lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1], ctx=f"flat K{K}")


def test_strides_unaligned_and_padded():
    rng = np.random.default_rng(5)
    Vp1 = 1025
    D = _small(rng, 3, 40, Vp1, stride=1028, pad=np.nan)
    L = np.array([40, 33, 12])
    cfg = F.config(8, beta=0.2)
    g_pad = gpu_decode(D, L, cfg, Vp1=Vp1)              # padded (16-B aligned rows)
    g_dense = gpu_decode(np.ascontiguousarray(D[:, :, :Vp1]), L, cfg)  # 4100-B rows (unaligned)
    for k in ("tokens", "num_tokens", "timestamps", "alignment"):
        assert np.array_equal(g_pad[k], g_dense[k])
    assert np.array_equal(g_pad["scores"].view(np.int32), g_dense["scores"].view(np.int32))
    o = oracle.decode_strided(np.ascontiguousarray(D[:, :, :Vp1]), Vp1, L, ocfg(cfg), None, None, NTH,
                              with_alignment=True)
    compare(g_dense, o)


def test_padding_is_never_read():
    """NaN in frames t >= L_b must not change anything (reading R16)."""
    rng = np.random.default_rng(6)
    D = _small(rng, 4, 50, 33)
    L = np.array([50, 10, 1, 0])
    cfg = F.config(8, beta=0.1)
    a = gpu_decode(D, L, cfg)
    Dn = D.copy()
    for b, l in enumerate(L):
        Dn[b, l:] = np.nan
    c = gpu_decode(Dn, L, cfg)
    for k in a:
        assert np.array_equal(a[k].view(np.int32), c[k].view(np.int32)), k


def test_batch_permutation_and_determinism(lm_pair, bt_pair):
    wl, D, L, _, _ = synth.workload_inputs("c4", B=16)
    cfg = wl_cfg(wl)
    a = gpu_decode(D, L, cfg, lm_pair[0], bt_pair[0])
    a2 = gpu_decode(D, L, cfg, lm_pair[0], bt_pair[0])
    for k in a:
        assert np.array_equal(a[k].view(np.int32), a2[k].view(np.int32)), k
    perm = np.random.default_rng(0).permutation(16)
    c = gpu_decode(D[perm], L[perm], cfg, lm_pair[0], bt_pair[0])
    for k in a:
        assert np.array_equal(a[k][perm].view(np.int32), c[k].view(np.int32)), k


def test_lengths_are_clamped_and_flagged():
    rng = np.random.default_rng(8)
    D = _small(rng, 3, 20, 9)
    Dt = torch.from_numpy(D).cuda()
    Lt = torch.tensor([25, -3, 20], dtype=torch.int32).cuda()
    cfg = F.config(4)
    ws = F.make_workspace(3, 20, 9, cfg)
    out = F.decode(Dt, Lt, cfg, workspace=ws)
    torch.cuda.synchronize()
    assert F.check(ws) == 3
    ref = gpu_decode(D, [20, 0, 20], cfg)
    assert np.array_equal(out["tokens"].cpu().numpy(), ref["tokens"])
    assert out["num_tokens"].cpu().numpy()[1] == 0


def test_all_minus_inf_frame_kills_the_utterance():
    D = np.full((1, 5, 4), -np.inf, np.float32)
    D[0, :2] = np.log(np.array([0.1, 0.2, 0.3, 0.4], np.float32))
    g = gpu_decode(D, [5], F.config(4))
    o = oracle.decode(D, [5], oracle.make_cfg(4, theta=12.0), nthreads=1, with_alignment=True)
    compare(g, o)
    assert g["num_tokens"][0] == 0 and g["scores"][0] == -np.inf


def test_empty_batch_and_zero_lengths(lm_pair):
    cfg = F.config(4, alpha_lm=0.5)
    D = np.zeros((2, 3, 1025), np.float32)
    g = gpu_decode(D, [0, 0], cfg, lm_pair[0])
    o = oracle.decode(D, [0, 0], ocfg(cfg), lm_pair[1], None, 1, with_alignment=True)
    compare(g, o)
    assert g["num_tokens"].tolist() == [0, 0]
    Dt = torch.zeros((0, 3, 1025), device="cuda")
    out = F.decode(Dt, torch.zeros(0, dtype=torch.int32, device="cuda"), cfg, lm_pair[0])
    assert out["tokens"].shape == (0, 3)


@pytest.mark.parametrize("streamed", [True, False])
@pytest.mark.parametrize("wname,B", [("c4", 8), ("c5", 24), ("c1", 1)])
def test_decode_host_end_to_end(lm_pair, bt_pair, wname, B, streamed, monkeypatch):
    """flexctc_decode_host (H2D in frame chunks overlapping the persistent kernel, or copy-then-
    decode) returns exactly what flexctc_decode returns on the same inputs: fixed lengths (2D
    chunk copies), ragged LibriSpeech-shaped lengths (pinned: the gather kernel), tiny c1."""
    if not streamed:
        monkeypatch.setenv("FLEXCTC_NO_STREAM_INPUT", "1")
    assert F.host_streaming() == streamed  # the B200 image supports stream memory operations
    wl, D, L, _, _ = synth.workload_inputs(wname, B=B)
    cfg = wl_cfg(wl, beam=min(wl.beam, 16))
    glm = lm_pair[0] if wl.lm else None
    gbt = bt_pair[0] if wl.boost else None
    Dp = torch.from_numpy(np.ascontiguousarray(D)).pin_memory()
    Lp = torch.from_numpy(L.astype(np.int32)).pin_memory()
    for _ in range(2):  # the second call reuses the per-thread copy stream
        out = F.decode_host(Dp, Lp, cfg, glm, gbt)
        g = gpu_decode(D, L, cfg, glm, gbt)
        assert np.array_equal(out["num_tokens"].numpy(), g["num_tokens"])
        assert np.array_equal(out["tokens"].numpy(), g["tokens"])
        assert np.array_equal(out["timestamps"].numpy(), g["timestamps"])
        assert np.array_equal(out["scores"].numpy().view(np.int32), g["scores"].view(np.int32))


def test_decode_host_ragged_pageable(lm_pair, bt_pair):
    """Ragged lengths from a pageable (not device-mapped) host buffer: the streamed path falls back
    from the gather kernel to 2D copies of runs of live utterances; same outputs as flexctc_decode."""
    assert F.host_streaming()
    wl, D, L, _, _ = synth.workload_inputs("c5", B=24)
    cfg = wl_cfg(wl, beam=16)
    out = F.decode_host(np.ascontiguousarray(D), L.astype(np.int32), cfg, lm_pair[0], bt_pair[0])
    g = gpu_decode(D, L, cfg, lm_pair[0], bt_pair[0])
    assert np.array_equal(out["tokens"].numpy(), g["tokens"])
    assert np.array_equal(out["timestamps"].numpy(), g["timestamps"])
    assert np.array_equal(out["scores"].numpy().view(np.int32), g["scores"].view(np.int32))


def test_decode_refuses_host_memory_through_abi():
    import ctypes
    from paper_2508_07315_b200 import flexctc as FX
    D = np.zeros((1, 2, 3), np.float32)
    L = np.ones(1, np.int32)
    cfg = F.config(2)
    ws = F.make_workspace(1, 2, 3, cfg)
    o = [torch.empty(2, dtype=torch.int32, device="cuda"), torch.empty(1, dtype=torch.int32, device="cuda"),
         torch.empty(1, device="cuda")]
    st = FX.lib.flexctc_decode(D.ctypes.data_as(ctypes.c_void_p), 6, 3, L.ctypes.data_as(ctypes.c_void_p), 1, 2, 3,
                               ctypes.byref(cfg), None, None, ctypes.c_void_p(ws.buf.data_ptr()), ws.nbytes, None,
                               ctypes.c_void_p(o[0].data_ptr()), ctypes.c_void_p(o[1].data_ptr()),
                               ctypes.c_void_p(o[2].data_ptr()), None, None)
    assert st == 1 and "no CPU path" in FX.last_error()


# ------------------------------------------------------------------------ invariants at full size

def _round_f32(x: Fraction) -> np.float32:
    f = np.float32(float(x))
    best = f
    for c in (np.nextafter(f, np.float32(-np.inf)), np.nextafter(f, np.float32(np.inf))):
        if abs(Fraction(float(c)) - x) < abs(Fraction(float(best)) - x):
            best = c
    return best


def _fmaf(a, b, c) -> np.float32:
    return _round_f32(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def test_eq1_replay_max_mode_c5(lm_pair, bt_pair):
    """Max mode: the returned score equals the canonical fp32 replay of Eq. (1) along the returned
    alignment (SURVEY §8(c) backtrace invariant) — checks the c5 GPU output at full size, every
    utterance, without running the oracle's search."""
    wl, D, L, _, _ = synth.workload_inputs("c5")
    cfg = wl_cfg(wl, merge_mode=1)
    g = gpu_decode(D, L, cfg, lm_pair[0], bt_pair[0])
    olm, obt = lm_pair[1], bt_pair[1]
    blank = wl.V
    f32 = np.float32
    for b in range(0, wl.B, 7):
        al = g["alignment"][b, :L[b]]
        s, prev, prefix = f32(0.0), blank, []
        for t, a in enumerate(al):
            s = f32(s + D[b, t, a])
            if a != blank and a != prev:
                s = f32(s + f32(cfg.beta))
                s = _fmaf(f32(cfg.alpha_lm), f32(olm.logp(prefix, int(a), f32=True)), s)
                s = _fmaf(f32(cfg.alpha_bt), f32(obt.delta(prefix, int(a), f32=True)), s)
                prefix.append(int(a))
            prev = a
        s = _fmaf(f32(cfg.alpha_lm), f32(olm.logp(prefix, -1, f32=True)), s)
        assert prefix == list(g["tokens"][b, :g["num_tokens"][b]])
        assert f32(g["scores"][b]) == s, (b, g["scores"][b], s)


@pytest.mark.parametrize("wname,nbest,mode", [("c1", 4, 0), ("c2", 3, 1), ("c3", 16, 0), ("c4", 5, 0), ("c4", 16, 1)])
def test_nbest_vs_oracle(lm_pair, bt_pair, wname, nbest, mode):
    """flexctc_decode_nbest (SPEC --nbest): every utterance's ranked final
    hypotheses (R15 merge, (score desc, slot asc)) equal the oracle's, row 0 equals flexctc_decode."""
    wl, D, L, _, _ = synth.workload_inputs(wname, B=6 if wname != "c1" else None)
    cfg = wl_cfg(wl, merge_mode=mode)
    glm = lm_pair[0] if wl.lm else None
    gbt = bt_pair[0] if wl.boost else None
    Dt, Lt = torch.from_numpy(np.ascontiguousarray(D)).cuda(), torch.from_numpy(L.astype(np.int32)).cuda()
    g = F.decode_nbest(Dt, Lt, cfg, nbest, glm, gbt)
    one = F.decode(Dt, Lt, cfg, glm, gbt)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in g.items()}
    one = {k: v.cpu().numpy() for k, v in one.items()}
    assert np.array_equal(g["tokens"][:, 0], one["tokens"]) and np.array_equal(g["num_tokens"][:, 0], one["num_tokens"])
    assert np.array_equal(g["timestamps"][:, 0], one["timestamps"])
    assert np.array_equal(g["scores"][:, 0].view(np.int32), one["scores"].view(np.int32))
    for b in range(D.shape[0]):
        ref = oracle.decode_nbest(D[b].astype(np.float64), ocfg(cfg), lm_pair[1] if wl.lm else None,
                                  bt_pair[1] if wl.boost else None, L=int(L[b]), f32=True)
        for r in range(nbest):
            n = int(g["num_tokens"][b, r])
            if r < len(ref):
                toks, sc = ref[r]
                assert tuple(g["tokens"][b, r, :n]) == toks, (b, r)
                assert (g["tokens"][b, r, n:] == -1).all()
                if mode == 1:
                    assert np.float32(g["scores"][b, r]) == np.float32(sc), (b, r)
                assert abs(float(g["scores"][b, r]) - sc) <= TOL, (b, r, float(g["scores"][b, r]), sc)
            else:
                assert n == 0 and g["scores"][b, r] == -np.inf


def test_nbest_rejects_bad_n():
    Dt = torch.zeros((1, 4, 5), device="cuda")
    Lt = torch.full((1,), 4, dtype=torch.int32, device="cuda")
    with pytest.raises(F.FlexCTCError):
        F.decode_nbest(Dt, Lt, F.config(4), 5)
    with pytest.raises(F.FlexCTCError):
        F.decode_nbest(Dt, Lt, F.config(4), 0)
