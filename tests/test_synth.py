"""The seeded input generators: deterministic, shaped like the paper's workloads."""
import numpy as np

import synth


def test_workload_shapes_and_determinism():
    wl, D, L, arpa, ph = synth.workload_inputs("c1")
    assert D.shape == (1, 50, 129) and L.tolist() == [50] and arpa is None and ph is None
    _, D2, _, _, _ = synth.workload_inputs("c1")
    assert np.array_equal(D, D2)
    # log-softmax rows
    assert np.allclose(np.exp(D[0].astype(np.float64)).sum(-1), 1.0, atol=1e-4)


def test_c4_statistics():
    wl, D, L, arpa, ph = synth.workload_inputs("c4", B=8)
    assert D.shape == (8, 400, 1025) and (L == 400).all() and len(ph) == 1000
    blank_frac = (D.argmax(-1) == 1024).mean()
    assert 0.7 < blank_frac < 0.9  # peaky CTC: mostly blank frames (0.16 tokens/frame)


def test_librispeech_lengths():
    wl = synth.WORKLOADS["c5"]
    L = synth.lengths(wl)
    assert L.shape == (512,) and L.max() <= 875 and L.min() >= 32
    assert 150 < L.mean() < 210  # mean 7.42 s at 40 ms


def test_phrases_distinct_lengths():
    ph = synth.phrases(1024)
    assert len(set(ph)) == 1000 and all(2 <= len(p) <= 5 for p in ph)


def test_lpt_inputs_pad_value():
    wl = synth.WORKLOADS["c5"]
    L = np.array([10, 3], dtype=np.int32)
    D, _ = synth.logprobs(2, 12, 16, L, 5, pad_value=np.nan)
    assert np.isnan(D[1, 3:]).all() and not np.isnan(D[0, :10]).any()
