"""Pins for the oracle (CPU only): the oracle is checked against what the paper and the
mathematics fix, never against itself (SURVEY.md §8(c) "Pins")."""
import math
import os

import numpy as np
import pytest
import torch

import oracle
from tests.conftest import GOLDEN
from tests.exact.arpa_py import ArpaPy
from tests.exact.boost_py import BoostPy
from tests.exact.ctc_exact import brute_force, ctc_forward, greedy
from tests.exact.exhaustive import exhaustive

INF = float("inf")


def _rand_logprobs(rng, T, Vp1, scale=1.5):
    x = rng.standard_normal((T, Vp1)) * scale
    return x - np.log(np.exp(x).sum(1, keepdims=True))


# ---------------------------------------------------------------- worked examples (SPEC)

def test_worked_T2_example(golden):
    g = golden["decode"]["worked_T2"]
    D = np.log(np.array(g["D"]))
    res = oracle.decode_nbest(D, oracle.make_cfg(4))
    assert res[0][0] == tuple(g["lse"]["best"])
    assert res[0][1] == pytest.approx(g["lse"]["best_score"], abs=1e-12)
    assert res[1][0] == tuple(g["lse"]["runner_up"])
    assert res[1][1] == pytest.approx(g["lse"]["runner_up_score"], abs=1e-12)
    resm = oracle.decode_nbest(D, oracle.make_cfg(4, merge_mode=1))
    assert resm[0][0] == tuple(g["max"]["best"])
    assert resm[0][1] == pytest.approx(g["max"]["best_score"], abs=1e-12)


def test_worked_T2_fp32_path(golden):
    g = golden["decode"]["worked_T2"]
    D = np.log(np.array(g["D"], dtype=np.float64)).astype(np.float32)[None]
    out = oracle.decode(D, [2], oracle.make_cfg(4))
    assert out["num_tokens"][0] == 1 and out["tokens"][0, 0] == 0
    assert out["scores"][0] == pytest.approx(g["lse"]["best_score"], abs=1e-6)


def test_theta_prune_example(golden):
    g = golden["decode"]["theta_prune"]
    D = np.array(g["D"])
    assert len(oracle.decode_nbest(D, oracle.make_cfg(2, theta=g["theta"]))) == g["n_alive"]
    assert len(oracle.decode_nbest(D, oracle.make_cfg(2, theta=INF))) == 2


def test_greedy_example(golden):
    g = golden["decode"]["greedy_T2"]
    D = np.log(np.array(golden["decode"]["worked_T2"]["D"]))
    res = oracle.decode_nbest(D, oracle.make_cfg(1))
    assert res[0][0] == tuple(g["tokens"])
    assert res[0][1] == pytest.approx(g["score"], abs=1e-12)


# ---------------------------------------------------------------- K = 1 == greedy

def test_beam1_equals_greedy_random():
    rng = np.random.default_rng(1)
    for trial in range(200):
        B = int(rng.integers(1, 9))
        T = int(rng.integers(1, 51))
        Vp1 = int(rng.integers(2, 17))
        D = np.stack([_rand_logprobs(rng, T, Vp1, 2.0) for _ in range(B)]).astype(np.float32)
        L = rng.integers(1, T + 1, B)
        out = oracle.decode(D, L, oracle.make_cfg(1), nthreads=2)
        for b in range(B):
            toks, score, _ = greedy(D[b, :L[b]], Vp1 - 1)
            n = out["num_tokens"][b]
            assert tuple(out["tokens"][b, :n]) == toks, (trial, b)
            assert out["scores"][b] == np.float32(score), (trial, b)


# ---------------------------------------------------------------- exact CTC (brute force, forward, ctc_loss)

@pytest.mark.parametrize("T,Vp1", [(1, 2), (2, 3), (3, 3), (4, 3), (5, 3), (6, 3), (3, 4), (4, 4), (5, 4), (6, 4),
                                   (3, 5), (4, 5), (5, 5)])
@pytest.mark.parametrize("mode", ["lse", "max"])
def test_full_beam_equals_brute_force(T, Vp1, mode):
    """θ = ∞, no fusion, K = V'^T (>= live states × V' at every frame): every transcript's score
    is exact (SURVEY §8(c) pin 1)."""
    rng = np.random.default_rng(100 * T + Vp1)
    K = Vp1 ** T
    for _ in range(3):
        D = _rand_logprobs(rng, T, Vp1)
        bf = brute_force(D, Vp1 - 1, mode)
        res = dict(oracle.decode_nbest(D, oracle.make_cfg(K, merge_mode=0 if mode == "lse" else 1)))
        assert set(res) == set(bf)
        for y, s in bf.items():
            assert res[y] == pytest.approx(s, abs=1e-10), y


def test_brute_force_equals_ctc_forward_and_ctc_loss():
    """Pins the brute-force checker itself against the textbook forward algorithm and the
    library routine torch.nn.functional.ctc_loss (which returns -log P(y|x))."""
    rng = np.random.default_rng(5)
    for _ in range(20):
        T, Vp1 = int(rng.integers(1, 6)), int(rng.integers(2, 5))
        D = _rand_logprobs(rng, T, Vp1)
        bf = brute_force(D, Vp1 - 1)
        for y, s in bf.items():
            assert ctc_forward(D, y, Vp1 - 1) == pytest.approx(s, abs=1e-10)
            if len(y) == 0:
                continue
            lp = torch.tensor(D, dtype=torch.float64)[:, None, :]
            loss = torch.nn.functional.ctc_loss(lp, torch.tensor([list(y)]), torch.tensor([T]),
                                                torch.tensor([len(y)]), blank=Vp1 - 1, reduction="none")
            assert -float(loss[0]) == pytest.approx(s, abs=1e-9)


def test_full_beam_matches_ctc_loss_t6():
    T, Vp1 = 6, 4
    rng = np.random.default_rng(9)
    D = _rand_logprobs(rng, T, Vp1)
    res = oracle.decode_nbest(D, oracle.make_cfg(Vp1 ** T))
    for y, s in res[:20]:
        if not y:
            continue
        lp = torch.tensor(D)[:, None, :]
        loss = torch.nn.functional.ctc_loss(lp, torch.tensor([list(y)]), torch.tensor([T]), torch.tensor([len(y)]),
                                            blank=Vp1 - 1, reduction="none")
        assert s == pytest.approx(-float(loss[0]), abs=1e-9)


# ---------------------------------------------------------------- LM fixtures

@pytest.mark.parametrize("fx,path", [("lm_2gram", "arpa_2gram.arpa"), ("lm_3gram", "arpa_3gram.arpa")])
def test_lm_fixture_values(golden, fx, path):
    g = golden[fx]
    syms = g["symbols"]
    lm = oracle.LM(os.path.join(GOLDEN, path), len(syms), syms)
    py = ArpaPy(os.path.join(GOLDEN, path))
    idx = {s: i for i, s in enumerate(syms)}
    for e in g["logp"]:
        hist = [idx[s] for s in e["hist"]]
        w = -1 if e["w"] == "</s>" else idx[e["w"]]
        assert lm.logp(hist, w) == pytest.approx(e["value"], abs=1e-7), e
        assert lm.logp(hist, w, f32=True) == pytest.approx(e["value"], abs=2e-6), e
        assert py.logp(["<s>"] + e["hist"], e["w"]) == pytest.approx(e["value"], abs=1e-7), e
    for e in g["seq"]:
        assert lm.seq([idx[s] for s in e["tokens"]]) == pytest.approx(e["value"], abs=1e-7), e
        assert py.seq(e["tokens"]) == pytest.approx(e["value"], abs=1e-7), e


def test_lm_errors(tmp_path):
    p = tmp_path / "bad.arpa"
    p.write_text("\\data\\\nngram 1=2\n\n\\1-grams:\n-1.0\t</s>\n\\end\\\n")
    with pytest.raises(ValueError, match="count mismatch"):
        oracle.LM(str(p), 1)
    p.write_text("\\data\\\nngram 1=1\n\n\\1-grams:\n-1.0\ta\n\\end\\\n")
    with pytest.raises(ValueError, match="</s>"):
        oracle.LM(str(p), 1, ["a"])
    p.write_text("\\data\\\nngram 1=1\n\n\\1-grams:\n-1.0\t</s>\n")
    with pytest.raises(ValueError, match="end"):
        oracle.LM(str(p), 1)
    p.write_text("\\data\\\nngram 1=2\n\n\\1-grams:\n-1.0\t</s>\n-1.0\ta\n\\end\\\n")
    with pytest.raises(ValueError, match="not in LM"):
        oracle.LM(str(p), 2, ["a", "zz"])


# ---------------------------------------------------------------- boosting fixtures

def test_boost_fixture_values(golden):
    g = golden["boost"]
    for e in g["cases"]:
        bt = oracle.Boost(e["phrases"], e["w"], 16)
        assert bt.delta(e["prefix"], e["token"]) == pytest.approx(e["delta"], abs=1e-12), e
        assert bt.delta(e["prefix"], e["token"], f32=True) == e["delta"], e
        py = BoostPy(e["phrases"], e["w"])
        u = 0
        for a in e["prefix"]:
            u = py.step(u, a)
        assert py.delta(u, e["token"])[0] == pytest.approx(e["delta"], abs=1e-12), e
    for e in g["U"]:
        assert oracle.Boost(e["phrases"], e["w"], 16).U(e["prefix"]) == pytest.approx(e["U"]), e
    for e in g["transition_depth"]:
        assert oracle.Boost(e["phrases"], 1.0, 16).state_depth(e["prefix"]) == e["depth"], e
    for e in g["sums"]:
        bt = oracle.Boost(e["phrases"], e["w"], 16)
        tot = sum(bt.delta(e["stream"][:i], e["stream"][i]) for i in range(len(e["stream"])))
        assert tot == pytest.approx(e["total"], abs=1e-12), e
        assert BoostPy(e["phrases"], e["w"]).total(e["stream"])[0] == pytest.approx(e["total"], abs=1e-12), e


def test_boost_naive_equals_aho_corasick_random():
    """Naive longest-suffix matching (oracle) == Aho-Corasick transition (tests/exact)."""
    rng = np.random.default_rng(3)
    for trial in range(60):
        V = int(rng.integers(2, 7))
        n = int(rng.integers(1, 8))
        phrases = [list(rng.integers(0, V, int(rng.integers(1, 5)))) for _ in range(n)]
        w = float(rng.uniform(0.2, 2.0))
        bt = oracle.Boost(phrases, w, V)
        py = BoostPy(phrases, w)
        stream = list(rng.integers(0, V, 40))
        u, tel = 0, 0.0
        for i, a in enumerate(stream):
            d_py, v = py.delta(u, int(a))
            assert bt.delta(stream[:i], int(a)) == pytest.approx(d_py, abs=1e-12)
            assert bt.state_depth(stream[:i + 1]) == py.depth[v]
            assert bt.U(stream[:i + 1]) == pytest.approx(py.U[v], abs=1e-12)
            tel += d_py
            u = v
        # telescoping: Σ deltas = committed total + U(end)  => Σ - U(end) = committed >= 0
        assert tel - py.U[u] >= -1e-9


def test_boost_errors():
    with pytest.raises(ValueError):
        oracle.Boost([], 1.0, 4)
    with pytest.raises(ValueError):
        oracle.Boost([[]], 1.0, 4)
    with pytest.raises(ValueError):
        oracle.Boost([[1, 4]], 1.0, 4)  # 4 == blank for V=4


# ---------------------------------------------------------------- Eq. (1) exactness with LM, BT, β

@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("retract", [0, 1])
def test_full_beam_equals_exhaustive_with_fusion(mode, retract):
    """With θ = ∞ and K = V'^T, every transcript's score = combine(acoustic) + α_LM·seq(y) +
    α_BT·Σ deltas(y) + β|y| (SURVEY §8(c) pin 2), on the 3-gram fixture (a, b, c; blank = 3)."""
    syms = ["a", "b", "c"]
    path = os.path.join(GOLDEN, "arpa_3gram.arpa")
    lm = oracle.LM(path, 3, syms)
    py = ArpaPy(path)
    phrases = [[0, 1], [1, 2], [0, 1, 2], [2, 2, 0]]
    bt = oracle.Boost(phrases, 0.7, 3)
    bpy = BoostPy(phrases, 0.7)
    rng = np.random.default_rng(11 + mode + 2 * retract)
    Vp1 = 4
    for T in [1, 2, 3, 4, 5]:
        D = _rand_logprobs(rng, T, Vp1)
        cfg = oracle.make_cfg(Vp1 ** T, alpha_lm=0.6, alpha_bt=0.8, beta=0.3, merge_mode=mode, retract=retract)
        res = dict(oracle.decode_nbest(D, cfg, lm=lm, boost=bt))
        ex = exhaustive(D, Vp1 - 1, "lse" if mode == 0 else "max", alpha_lm=0.6, lm=py, symbols=syms,
                        alpha_bt=0.8, boost=bpy, beta=0.3, retract=bool(retract))
        assert set(res) == set(ex)
        for y, s in ex.items():
            assert res[y] == pytest.approx(s, abs=1e-10), (T, y)


def test_lm_empty_utterance_score():
    """L_b = 0 -> empty transcript with score α_LM·Final(<s>)."""
    lm = oracle.LM(os.path.join(GOLDEN, "arpa_2gram.arpa"), 2, ["a", "b"])
    D = np.zeros((3, 3))
    res = oracle.decode_nbest(D, oracle.make_cfg(2, alpha_lm=0.5), lm=lm, L=0)
    assert res == [((), pytest.approx(0.5 * -2.302585092994046, abs=1e-12))]


# ---------------------------------------------------------------- synthetic LM is a normalised backoff LM

@pytest.mark.slow
def test_synthetic_arpa_normalised():
    import synth
    path = synth.arpa_file(V=1024)
    lm = oracle.LM(path, 1024)
    assert lm.order == 4
    rng = np.random.default_rng(0)
    src = synth.MarkovSource(1024, synth.LM_SEED)
    hists = [[]] + [list(src.sequences(rng, 1, int(n))[0]) for n in [1, 2, 3, 5, 8]] + \
            [list(rng.integers(0, 1024, 3))]
    for h in hists:
        tot = sum(math.exp(lm.logp(h, w)) for w in range(1024)) + math.exp(lm.logp(h, -1))
        assert tot == pytest.approx(1.0, abs=1e-3), h


# ----------------------------------------------------------------- input side: bf16 log-softmax
# SURVEY §8(f) NEXT 4 (log-softmax of bf16 logits fused into the frame read); DESIGN.md reading
# R25 fixes the arithmetic: exact bf16 values, fp64 max / sum / log, one rounding to fp32.

def _bf16_bits(x):
    """Round-to-nearest-even fp32 -> bf16 bit patterns (uint16)."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def _bf16_value(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def test_log_softmax_bf16_hand_cases():
    # logits exactly representable in bf16: [0, 1, -2, 0.5]; lse = ln(1 + e + e^-2 + e^0.5)
    bits = _bf16_bits(np.array([[0.0, 1.0, -2.0, 0.5]], np.float32))
    out = oracle.log_softmax_bf16(bits)
    lse = math.log(1 + math.e + math.exp(-2.0) + math.exp(0.5))
    assert out.tolist() == [[float(np.float32(v - lse)) for v in (0.0, 1.0, -2.0, 0.5)]]
    # uniform logits: every output is -ln(V') rounded once, whatever the common value
    for c in (0.0, 7.5, -13.25):
        bits = _bf16_bits(np.full((2, 1025), c, np.float32))
        out = oracle.log_softmax_bf16(bits)
        assert (out == np.float32(-math.log(1025))).all()


def test_log_softmax_bf16_matches_numpy_fp64():
    rng = np.random.default_rng(3)
    x = (rng.standard_normal((64, 1025)) * 3.0).astype(np.float32)
    x[:, 17] += 15.0  # a peaky column, as the synthetic CTC rows
    bits = _bf16_bits(x)
    v = _bf16_value(bits)
    m = v.max(-1, keepdims=True)
    ref = (v - (m + np.log(np.exp(v - m).sum(-1, keepdims=True)))).astype(np.float32)
    out = oracle.log_softmax_bf16(bits)
    # the fp64 sums differ only in summation order (~1e-16 relative): the rounded fp32 outputs
    # agree exactly except at a rounding boundary, and never by more than one ulp
    ulp = np.spacing(np.abs(ref))
    assert (np.abs(out.astype(np.float64) - ref) <= ulp).all()
    assert (out == ref).mean() > 0.9999
    assert np.allclose(np.exp(out.astype(np.float64)).sum(-1), 1.0, atol=1e-5)


# ---------------------------------------------------------------- timestamps and tie rules (round 2)

def _peaky(align, Vp1, p):
    """log-probs putting p on align[t] and (1-p)/(V'-1) on every other label of frame t"""
    D = np.full((len(align), Vp1), (1.0 - p) / (Vp1 - 1))
    D[np.arange(len(align)), align] = p
    return np.log(D)


@pytest.mark.parametrize("mode", [0, 1])
def test_timestamps_hand_fixtures(golden, mode):
    """R20 timestamps = emission frames of the survivor's alignment (tests/golden 'timestamps')."""
    g = golden["decode"]["timestamps"]
    for case in g["cases"]:
        D = _peaky(case["align"], 3, g["p_target"]).astype(np.float32)[None]
        out = oracle.decode(D, [len(case["align"])], oracle.make_cfg(4, merge_mode=mode), with_alignment=True)
        n = int(out["num_tokens"][0])
        assert out["tokens"][0, :n].tolist() == case["tokens"]
        assert out["timestamps"][0, :n].tolist() == case["timestamps"]
        assert out["alignment"][0, :len(case["align"])].tolist() == case["align"]
        assert (out["timestamps"][0, n:] == -1).all() and (out["tokens"][0, n:] == -1).all()


def test_timestamps_match_planted_spikes():
    """Weak pin of R20 (SURVEY §8(c) 'Unpinned'): on peaky synthetic data the best path emits its
    tokens at the planted spike frames. 8 c2-shaped utterances (V=1024, no fusion; competitor
    spikes cause some substitutions and insertions): the fraction of decoded tokens whose
    timestamp is a planted spike frame of the utterance must be >= 0.95, and the tokens that
    match the planted one at that frame must be >= 0.85 of all decoded tokens."""
    import synth
    wl = synth.WORKLOADS["c2"]
    L = synth.lengths(wl, 8, wl.seed)
    D, tr, frames = synth.logprobs(8, wl.T, wl.V, L, wl.seed, return_frames=True)
    out = oracle.decode(D, L, oracle.make_cfg(wl.beam, beta=wl.beta, theta=wl.theta), nthreads=8)
    at_spike = same = tot = 0
    for b in range(8):
        n = int(out["num_tokens"][b])
        planted = dict(zip(frames[b], tr[b]))
        for tok, ts in zip(out["tokens"][b, :n].tolist(), out["timestamps"][b, :n].tolist()):
            tot += 1
            at_spike += int(ts in planted)
            same += int(planted.get(ts) == tok)
    assert tot > 400
    assert at_spike / tot >= 0.95, at_spike / tot
    assert same / tot >= 0.85, same / tot


def test_topk_tie_rule(golden):
    """SPEC S:342 / R9: equal candidates -> the lower flat index enters the TopK (tests/golden 'topk_tie')."""
    g = golden["decode"]["topk_tie"]
    D = np.log(np.array(g["D"]))
    res = oracle.decode_nbest(D, oracle.make_cfg(g["beam"]))
    assert [list(t) for t, _ in res] == g["nbest_tokens"]
    assert res[0][1] == res[1][1]
    D32 = D.astype(np.float32)[None]
    out = oracle.decode(D32, [1], oracle.make_cfg(g["beam"]))
    assert out["tokens"][0, :int(out["num_tokens"][0])].tolist() == g["nbest_tokens"][0]


@pytest.mark.parametrize("mode", [0, 1])
def test_merge_tie_rule(golden, mode):
    """SPEC S:98 / R12, R14: equal-score members of a merge group -> the lower slot survives; its
    alignment decides the timestamps (tests/golden 'merge_tie')."""
    g = golden["decode"]["merge_tie"]
    D = np.log(np.array(g["D"], dtype=np.float64)).astype(np.float32)[None]
    out = oracle.decode(D, [2], oracle.make_cfg(g["beam"], merge_mode=mode), with_alignment=True)
    assert out["tokens"][0, :int(out["num_tokens"][0])].tolist() == g["tokens"]
    assert out["timestamps"][0, :1].tolist() == g["timestamps"]
    assert out["alignment"][0].tolist() == g["alignment"]
    want = math.log(0.5) + math.log(0.7) if mode == 1 else math.log(0.85)
    assert float(out["scores"][0]) == pytest.approx(want, abs=1e-6)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("fuse", [0, 1])
def test_full_beam_equals_path_enumeration(mode, fuse):
    """The path-level enumerator (every alignment scored on its own, then combined per transcript)
    agrees with the full beam, both for Alg. 1 and for the P:167 variant that scores every
    repeated emission with the LM / BT (fuse_repeats): the variant's extra terms depend only on
    (prefix, last label), so recombination stays exact."""
    from tests.exact.exhaustive import exhaustive_paths
    syms = ["a", "b", "c"]
    path = os.path.join(GOLDEN, "arpa_3gram.arpa")
    lm = oracle.LM(path, 3, syms)
    py = ArpaPy(path)
    phrases = [[0, 1], [1, 2], [0, 1, 2], [2, 2, 0], [1, 1]]
    bt = oracle.Boost(phrases, 0.7, 3)
    bpy = BoostPy(phrases, 0.7)
    rng = np.random.default_rng(23 + mode + 2 * fuse)
    Vp1 = 4
    for T in [1, 2, 3, 4, 5]:
        D = _rand_logprobs(rng, T, Vp1)
        cfg = oracle.make_cfg(Vp1 ** T, alpha_lm=0.6, alpha_bt=0.8, beta=0.3, merge_mode=mode, fuse_repeats=fuse)
        res = dict(oracle.decode_nbest(D, cfg, lm=lm, boost=bt))
        ex = exhaustive_paths(D, Vp1 - 1, "lse" if mode == 0 else "max", alpha_lm=0.6, lm=py, symbols=syms,
                              alpha_bt=0.8, boost=bpy, beta=0.3, fuse_repeats=bool(fuse))
        assert set(res) == set(ex)
        for y, s in ex.items():
            assert res[y] == pytest.approx(s, abs=1e-10), (T, y, fuse)
    if fuse:  # the variant changes scores of transcripts whose alignments repeat a token
        D = _rand_logprobs(np.random.default_rng(5), 3, Vp1)
        a = dict(oracle.decode_nbest(D, oracle.make_cfg(64, alpha_lm=0.6, fuse_repeats=1), lm=lm))
        b = dict(oracle.decode_nbest(D, oracle.make_cfg(64, alpha_lm=0.6, fuse_repeats=0), lm=lm))
        assert a[()] == b[()] and any(abs(a[y] - b[y]) > 1e-6 for y in a if y)


# ------------------------------------------------------ merge-before-TopK variant (reading R27)
# BJ north_star: "merges duplicate prefixes by prefix hash, selects the top-K"; Alg. 1
# selects first. merge_first = 1 recombines every (transcript, last label) group of the K·V'
# candidates before the TopK.

def test_merge_first_hand_fixture():
    """Hand-derived two-frame case (a = 0, b = 1, blank = 2; K = 2, lse, no fusion terms).
    Frame 0 from the empty beam: P(a) .5, P(b) .2, P(∅) .3 -> slots (a | a) .5 and (∅ | ∅) .3.
    Frame 1, P(a) .32, P(b) .4, P(∅) .28; candidates (probabilities):
      (a|a): .5·.32 = .16 (repeat) and .3·.32 = .096 (emission from ∅) -> group .256
      (ab|b): .5·.4 = .20;  (a|∅): .5·.28 = .14;  (b|b): .3·.4 = .12;  (∅|∅): .3·.28 = .084
    Merge first: the groups (a|a) .256 and (ab|b) .20 survive -> 1-best "a" at ln .256.
    Alg. 1 (TopK first): candidates .20 (ab|b) and .16 (a|a) survive -> 1-best "ab" at ln .20,
    "a" at ln .16 (the .096 member was cut before the merge)."""
    D = np.log(np.array([[0.5, 0.2, 0.3], [0.32, 0.4, 0.28]]))
    mf = dict(oracle.decode_nbest(D, oracle.make_cfg(2, merge_first=1)))
    tk = dict(oracle.decode_nbest(D, oracle.make_cfg(2)))
    assert set(mf) == {(0,), (0, 1)} and set(tk) == {(0,), (0, 1)}
    assert mf[(0,)] == pytest.approx(math.log(0.256), abs=1e-12)
    assert mf[(0, 1)] == pytest.approx(math.log(0.20), abs=1e-12)
    assert tk[(0,)] == pytest.approx(math.log(0.16), abs=1e-12)
    assert tk[(0, 1)] == pytest.approx(math.log(0.20), abs=1e-12)
    # max combiner: the (a|a) group scores its best member (.16) and ranks below (ab|b) .20
    mfx = dict(oracle.decode_nbest(D, oracle.make_cfg(2, merge_mode=1, merge_first=1)))
    assert mfx[(0,)] == pytest.approx(math.log(0.16), abs=1e-12)
    # θ-prune relative to the best GROUP: K = 3, θ = 0.6 keeps ∅ at frame 0 (ln(.5/.3) = .51) and
    # prunes b (.92); at frame 1 the cut is .256·e^-.6 = .1405, so (a|∅) .14 is dropped (it would
    # survive a cut relative to the best single candidate, .20·e^-.6 = .1098, and then add to "a"
    # in the final merge): "a" stays at ln .256, "ab" at ln .20
    mft = dict(oracle.decode_nbest(D, oracle.make_cfg(3, theta=0.6, merge_first=1)))
    assert set(mft) == {(0,), (0, 1)}
    assert mft[(0,)] == pytest.approx(math.log(0.256), abs=1e-12)
    assert mft[(0, 1)] == pytest.approx(math.log(0.20), abs=1e-12)


def _max_groups(T, Vp1):
    """Largest number of distinct (transcript, last label) pairs over the frames (brute force)."""
    import itertools
    blank, best = Vp1 - 1, 0
    for t in range(1, T + 1):
        keys = set()
        for a in itertools.product(range(Vp1), repeat=t):
            y, prev = [], blank
            for w in a:
                if w != blank and w != prev:
                    y.append(w)
                prev = w
            keys.add((tuple(y), a[-1]))
        best = max(best, len(keys))
    return best


@pytest.mark.parametrize("mode", [0, 1])
def test_merge_first_exact_with_group_sized_beam(mode):
    """Merge-first keeps every (transcript, last) group when K >= their number, so with θ = ∞ it
    equals the path enumeration already at K = max #groups (< K·V' candidates). Alg. 1 at the
    same K cuts candidates before merging and must deviate somewhere (the pin separates the two)."""
    from tests.exact.exhaustive import exhaustive_paths
    syms = ["a", "b", "c"]
    path = os.path.join(GOLDEN, "arpa_3gram.arpa")
    lm = oracle.LM(path, 3, syms)
    py = ArpaPy(path)
    phrases = [[0, 1], [1, 2], [0, 1, 2], [2, 2, 0], [1, 1]]
    bt = oracle.Boost(phrases, 0.7, 3)
    bpy = BoostPy(phrases, 0.7)
    rng = np.random.default_rng(77 + mode)
    Vp1 = 4
    deviates = False
    for T in [1, 2, 3, 4, 5]:
        D = _rand_logprobs(rng, T, Vp1)
        K = _max_groups(T, Vp1)
        kw = dict(alpha_lm=0.6, alpha_bt=0.8, beta=0.3, merge_mode=mode)
        res = dict(oracle.decode_nbest(D, oracle.make_cfg(K, merge_first=1, **kw), lm=lm, boost=bt))
        ex = exhaustive_paths(D, Vp1 - 1, "lse" if mode == 0 else "max", alpha_lm=0.6, lm=py, symbols=syms,
                              alpha_bt=0.8, boost=bpy, beta=0.3)
        assert set(res) == set(ex), T
        for y, s in ex.items():
            assert res[y] == pytest.approx(s, abs=1e-10), (T, y)
        alg1 = dict(oracle.decode_nbest(D, oracle.make_cfg(K, **kw), lm=lm, boost=bt))
        deviates |= set(alg1) != set(ex) or any(abs(alg1[y] - ex[y]) > 1e-9 for y in alg1)
    assert deviates


def test_merge_first_full_beam_equals_alg1():
    """With K >= K·V' candidates and θ = ∞ nothing is cut: both orders are exact and agree."""
    rng = np.random.default_rng(3)
    for T in [1, 2, 3, 4]:
        D = _rand_logprobs(rng, T, 3)
        a = dict(oracle.decode_nbest(D, oracle.make_cfg(3 ** T, merge_first=1)))
        b = dict(oracle.decode_nbest(D, oracle.make_cfg(3 ** T)))
        assert set(a) == set(b)
        for y in a:
            assert a[y] == pytest.approx(b[y], abs=1e-12)
