"""CPU tests of the product's C-ABI library: it loads, exports every declared symbol, and its
host-built LM / boost layouts answer queries bit-identically to the oracle's independent
evaluators (no GPU needed: the layouts are built on the host before upload)."""
import os
import re

import numpy as np
import pytest

import oracle
import paper_2508_07315_b200 as F
from paper_2508_07315_b200 import flexctc as FX
from tests.conftest import GOLDEN, ROOT


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "flexctc.h")).read()
    declared = set(re.findall(r"\b(flexctc_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(FX.lib, name), name
    assert set(FX.EXPORTS) == declared


def _walk(lm, hist):
    s = lm.info().start_state
    for w in hist:
        _, s = lm.host_query(s, w)
    return s


@pytest.mark.parametrize("path,syms", [("arpa_2gram.arpa", ["a", "b"]), ("arpa_3gram.arpa", ["a", "b", "c"])])
def test_lm_layout_equals_oracle_on_fixtures(path, syms):
    p = os.path.join(GOLDEN, path)
    lm = F.LM(p, len(syms), syms, device=-1)
    orc = oracle.LM(p, len(syms), syms)
    V = len(syms)
    import itertools
    for n in range(0, 5):
        for hist in itertools.product(range(V), repeat=n):
            s = _walk(lm, hist)
            for w in list(range(V)) + [-1]:
                got, _ = lm.host_query(s, w)
                want = orc.logp(list(hist), w, f32=True)
                assert np.float32(got) == np.float32(want), (hist, w, got, want)


def test_lm_layout_equals_oracle_on_synthetic_lm():
    import synth
    path = synth.arpa_file(V=1024)
    lm = F.LM(path, 1024, device=-1)
    info = lm.info()
    assert info.order == 4 and info.n_arcs > 500_000
    orc = oracle.LM(path, 1024)
    rng = np.random.default_rng(0)
    src = synth.MarkovSource(1024, synth.LM_SEED)
    n_checked = 0
    for trial in range(40):
        seq = list(src.sequences(rng, 1, int(rng.integers(0, 12)))[0]) if trial % 4 else list(rng.integers(0, 1024, 5))
        s = _walk(lm, seq)
        ws = list(rng.integers(0, 1024, 40)) + [-1] + list(src.sequences(rng, 1, 1)[0])
        for w in ws:
            got, _ = lm.host_query(s, int(w))
            want = orc.logp(seq, int(w), f32=True)
            assert np.float32(got) == np.float32(want), (seq, w, got, want)
            n_checked += 1
    assert n_checked > 1500


def _random_histories(rng, src, n):
    """Markov-source histories (the contexts decoding visits) mixed with uniform random ones."""
    out = []
    for i in range(n):
        k = int(rng.integers(0, 13))
        out.append(list(map(int, src.sequences(rng, 1, k)[0]))[:k] if i % 3 else list(map(int, rng.integers(0, 1024, k))))
    return out


def test_lm_layout_one_million_queries():
    """SURVEY §4 tier 2: 10^6 random (history, token) queries of the synthetic 4-gram through the
    product's state layout equal the oracle's direct ARPA evaluator bit for bit (fp32)."""
    import synth
    path = synth.arpa_file(V=1024)
    lm = F.LM(path, 1024, device=-1)
    orc = oracle.LM(path, 1024)
    rng = np.random.default_rng(5)
    src = synth.MarkovSource(1024, synth.LM_SEED)
    n = 0
    for hist in _random_histories(rng, src, 1000):
        s = _walk(lm, hist)
        succ = list(map(int, src.sequences(rng, 1, 24)[0]))  # likely continuations (arc hits)
        ws = np.concatenate([rng.integers(0, 1024, 975), np.array(succ[:24] + [-1])]).astype(np.int32)
        got, _ = lm.host_query_batch(np.full(ws.shape[0], s, np.int32), ws)
        want = orc.logp_many(hist, ws, f32=True).astype(np.float32)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (hist, ws[bad[:5]], got[bad[:5]], want[bad[:5]])
        n += ws.shape[0]
    assert n >= 1_000_000


def test_lm_upper_bound_is_valid():
    """The pre-prune bound ub(s) (flexctc_lm_host_bound) is >= max_w log P(w | s) over all 1024
    decoder tokens, on random states (a too-small ub would make the exact pre-prune drop a
    candidate); and it is not vacuous (within 1 nat of the max on most states)."""
    import synth
    lm = F.LM(synth.arpa_file(V=1024), 1024, device=-1)
    rng = np.random.default_rng(1)
    src = synth.MarkovSource(1024, synth.LM_SEED)
    allw = np.arange(1024, dtype=np.int32)
    tight = 0
    hists = _random_histories(rng, src, 300)
    for hist in hists:
        s = _walk(lm, hist)
        vals, _ = lm.host_query_batch(np.full(1024, s, np.int32), allw)
        ub, _ = lm.host_bound(s)
        assert float(ub) >= float(vals.max()), (hist, ub, vals.max())
        tight += (float(ub) - float(vals.max())) < 1.0
    assert tight > 0.9 * len(hists)


def _bt_walk(bt, seq):
    u = 0
    for a in seq:
        _, u, _ = bt.host_query(u, a)
    return u


def test_boost_layout_equals_oracle_fixtures(golden):
    for e in golden["boost"]["cases"]:
        bt = F.Boost(e["phrases"], e["w"], 16, device=-1)
        u = _bt_walk(bt, e["prefix"])
        d, _, _ = bt.host_query(u, e["token"])
        assert d == e["delta"], e
    for e in golden["boost"]["U"]:
        bt = F.Boost(e["phrases"], e["w"], 16, device=-1)
        u = _bt_walk(bt, e["prefix"])
        assert bt.host_query(u, 0)[2] == e["U"], e


def test_boost_layout_equals_oracle_random():
    rng = np.random.default_rng(7)
    for trial in range(40):
        V = int(rng.integers(2, 9))
        phrases = [list(map(int, rng.integers(0, V, int(rng.integers(1, 6))))) for _ in range(int(rng.integers(1, 10)))]
        w = float(np.float32(rng.uniform(0.1, 3.0)))
        bt = F.Boost(phrases, w, V, device=-1)
        orc = oracle.Boost(phrases, w, V)
        stream = list(map(int, rng.integers(0, V, 50)))
        u = 0
        for i, a in enumerate(stream):
            d, v, Uu = bt.host_query(u, a)
            assert np.float32(d) == np.float32(orc.delta(stream[:i], a, f32=True)), (trial, i)
            assert np.float32(Uu) == np.float32(orc.U(stream[:i], f32=True))
            u = v


def _sig_bit(a):
    return ((a * 0x9E3779B1) & 0xFFFFFFFF) >> 26


@pytest.mark.parametrize("synthetic", [False, True])
def test_boost_signature_shortcut_is_exact(synthetic):
    """The kernels serve a boost lookup (u, a) from the root row when a is outside u's exception
    signature: δ(u, a) = δ(root, a) and delta(u, a) = fl(delta(root, a) - U(u)) must then hold
    exactly, and the signature must cover every token whose transition differs from the root's."""
    import synth
    rng = np.random.default_rng(3)
    cases = []
    if synthetic:
        cases.append((synth.phrases(1024), 1.0, 1024))
    else:
        for _ in range(30):
            V = int(rng.integers(2, 12))
            ph = [list(map(int, rng.integers(0, V, int(rng.integers(1, 6))))) for _ in range(int(rng.integers(1, 12)))]
            cases.append((ph, float(np.float32(rng.uniform(0.1, 3.0))), V))
    for ph, w, V in cases:
        bt = F.Boost(ph, w, V, device=-1)
        N = bt.num_nodes()
        nodes = range(N) if N * V <= 200_000 else rng.choice(N, 150, replace=False)
        allw = np.arange(V, dtype=np.int32)
        d0, n0 = bt.host_query_batch(np.zeros(V, np.int32), allw)
        assert bt.host_signature(0) == 0
        for u in nodes:
            u = int(u)
            d, nx = bt.host_query_batch(np.full(V, u, np.int32), allw)
            Uu = np.float32(bt.host_query(u, 0)[2])
            sig = bt.host_signature(u)
            for a in range(V):
                if (sig >> _sig_bit(a)) & 1:
                    continue
                assert nx[a] == n0[a], (u, a)
                assert np.float32(d[a]) == np.float32(np.float32(d0[a]) - Uu), (u, a, d[a], d0[a], Uu)


def test_boost_synthetic_phrases_size():
    import synth
    ph = synth.phrases(1024)
    bt = F.Boost(ph, 1.0, 1024, device=-1)
    assert 2000 < bt.num_nodes() < 5000


def test_errors_are_reported(tmp_path):
    p = tmp_path / "bad.arpa"
    p.write_text("\\data\\\nngram 1=2\n\n\\1-grams:\n-1.0\t</s>\n\\end\\\n")
    with pytest.raises(F.FlexCTCError, match="PARSE.*count mismatch"):
        F.LM(str(p), 1, device=-1)
    p.write_text("\\data\\\nngram 1=2\nngram 2=1\n\n\\1-grams:\n-1.0\t</s>\n-1.0\ta\n\n\\2-grams:\n-0.5\tb a\n\\end\\\n")
    with pytest.raises(F.FlexCTCError, match="PARSE"):
        F.LM(str(p), 1, ["a"], device=-1)
    # prefix property: "a b c" listed without "a b"
    p.write_text("\\data\\\nngram 1=4\nngram 2=1\nngram 3=1\n\n\\1-grams:\n-1\t</s>\n-1\ta\n-1\tb\n-1\tc\n\n"
                 "\\2-grams:\n-0.5\tb c\n\n\\3-grams:\n-0.1\ta b c\n\\end\\\n")
    with pytest.raises(F.FlexCTCError, match="unlisted context"):
        F.LM(str(p), 3, ["a", "b", "c"], device=-1)
    p.write_text("\\data\\\nngram 1=2\n\n\\1-grams:\n-1.0\t</s>\n-1.0\ta\n\\end\\\n")
    with pytest.raises(F.FlexCTCError, match="VOCAB_BIND"):
        F.LM(str(p), 2, ["a", "zz"], device=-1)
    with pytest.raises(F.FlexCTCError, match="IO"):
        F.LM(str(tmp_path / "missing.arpa"), 2, device=-1)
    with pytest.raises(F.FlexCTCError, match="INVALID_ARG"):
        F.Boost([[1, 4]], 1.0, 4, device=-1)
    with pytest.raises(F.FlexCTCError, match="INVALID_ARG"):
        F.Boost([[]], 1.0, 4, device=-1)
    with pytest.raises(F.FlexCTCError, match="INVALID_ARG"):
        F.Boost([[1]], 0.0, 4, device=-1)


def test_decode_refuses_cpu_tensors():
    import torch
    D = torch.zeros((1, 2, 3))
    L = torch.ones(1, dtype=torch.int32)
    with pytest.raises(F.FlexCTCError, match="no CPU path"):
        F.decode(D, L, F.config(2))


def test_workspace_bytes():
    cfg = F.config(16)
    n = F.workspace_bytes(64, 400, 1025, cfg)
    assert n >= 64 * 400 * 16 * 3
