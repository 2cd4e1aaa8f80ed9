"""GPU parity of the merge-before-TopK variant (config merge_first = 1, merge_first_kernel.cu;
DESIGN.md reading R27) against the oracle's merge_first flag, which is pinned
in tests/test_oracle_pins.py (hand fixture + exactness at K = max #groups)."""
import math
import os

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
from tests.test_gpu_parity import gpu_decode, run_pair, wl_cfg  # noqa: E402


def _small_fusion():
    syms = ["a", "b", "c"]
    arpa = os.path.join(GOLDEN, "arpa_3gram.arpa")
    phrases = [[0, 1], [1, 2, 0], [2, 2]]
    return (F.LM(arpa, 3, syms, device=0), oracle.LM(arpa, 3, syms), F.Boost(phrases, 0.9, 3, device=0),
            oracle.Boost(phrases, 0.9, 3))


def test_hand_fixture_on_gpu():
    """The two-frame fixture of test_merge_first_hand_fixture: 1-best "a" at ln .256 (Alg. 1: "ab")."""
    D = np.log(np.array([[[0.5, 0.2, 0.3], [0.32, 0.4, 0.28]]])).astype(np.float32)
    L = [2]
    g = gpu_decode(D, L, F.config(2, theta=float("inf"), merge_first=1))
    assert int(g["num_tokens"][0]) == 1 and g["tokens"][0, 0] == 0
    assert abs(float(g["scores"][0]) - math.log(0.256)) < 1e-6
    a = gpu_decode(D, L, F.config(2, theta=float("inf")))
    assert a["tokens"][0, :2].tolist() == [0, 1]
    g3 = gpu_decode(D, L, F.config(3, theta=0.6, merge_first=1))
    assert abs(float(g3["scores"][0]) - math.log(0.256)) < 1e-6


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("K,theta", [(2, float("inf")), (4, 3.0), (8, float("inf")), (3, 1.5)])
def test_small_vocab_with_fusion(mode, K, theta):
    """V' = 4 (the golden 3-gram LM + phrases), ragged lengths incl. 0 and 1, seeded peaky and
    flat frames; bit-identical scores in max mode."""
    glm, olm, gbt, obt = _small_fusion()
    rng = np.random.default_rng(100 + 7 * K + mode)
    B, T = 12, 30
    D = synth.random_logprobs(rng, B, T, 4, peak=2.5).astype(np.float32)
    L = rng.integers(0, T + 1, B).astype(np.int32)
    L[0], L[1] = 0, 1
    cfg = F.config(K, alpha_lm=0.5, alpha_bt=1.0, beta=0.3, theta=theta, merge_mode=mode, merge_first=1)
    run_pair(D, L, cfg, glm, olm, gbt, obt, ctx=f"mf small K{K} mode{mode}")


@pytest.mark.parametrize("fuse", [0, 1])
def test_small_vocab_no_lm_and_fuse_repeats(fuse):
    rng = np.random.default_rng(9 + fuse)
    B, T, Vp1 = 10, 40, 9
    D = synth.random_logprobs(rng, B, T, Vp1, peak=1.5).astype(np.float32)
    L = rng.integers(1, T + 1, B).astype(np.int32)
    run_pair(D, L, F.config(6, beta=0.4, theta=6.0, merge_first=1, fuse_repeats=fuse), ctx=f"mf nolm fuse{fuse}")
    glm, olm, gbt, obt = _small_fusion()
    D4 = synth.random_logprobs(rng, B, T, 4, peak=1.5).astype(np.float32)
    run_pair(D4, L, F.config(5, alpha_lm=0.7, alpha_bt=0.6, beta=0.2, theta=8.0, merge_first=1, fuse_repeats=fuse),
             glm, olm, gbt, obt, ctx=f"mf fusion fuse{fuse}")


@pytest.mark.parametrize("wname,B,K,mode", [("c1", 4, 4, 0), ("c1", 4, 1, 0), ("c4", 4, 16, 0), ("c4", 3, 16, 1),
                                            ("c4", 3, 1, 1), ("c3", 3, 8, 0), ("c5", 2, 32, 0)])
def test_paper_shapes(lm_pair, bt_pair, wname, B, K, mode):
    """Paper-shaped utterances (V' = 129 / 1025, the synthetic 4-gram LM and 1000 phrases where the
    workload has them) through the variant."""
    wl, D, L, _, _ = synth.workload_inputs(wname, B=B)
    glm, olm = (lm_pair[0], lm_pair[1]) if wl.lm else (None, None)
    gbt, obt = (bt_pair[0], bt_pair[1]) if wl.boost else (None, None)
    run_pair(D, L, wl_cfg(wl, beam=K, merge_mode=mode, merge_first=1), glm, olm, gbt, obt,
             ctx=f"mf {wname} K{K} mode{mode}")


@pytest.mark.parametrize("K,theta,mode", [(64, float("inf"), 0), (128, 6.0, 1), (256, 8.0, 0)])
def test_large_beams(K, theta, mode):
    """K = 64 .. 256 (the buffer cut with hundreds of groups per frame), V' = 33, flat frames."""
    rng = np.random.default_rng(K + mode)
    B, T, Vp1 = 4, 60, 33
    D = synth.random_logprobs(rng, B, T, Vp1, peak=1.0).astype(np.float32)
    L = rng.integers(30, T + 1, B).astype(np.int32)
    run_pair(D, L, F.config(K, beta=0.2, theta=theta, merge_mode=mode, merge_first=1), ctx=f"mf K{K}")


def test_flag_is_live_and_nbest_refused(lm_pair, bt_pair):
    # flat frames and a small beam: members of one group fall on both sides of Alg. 1's TopK cut
    rng = np.random.default_rng(4)
    D = synth.random_logprobs(rng, 8, 30, 9, peak=1.0).astype(np.float32)
    L = np.full(8, 30, np.int32)
    a = gpu_decode(D, L, F.config(3, theta=float("inf"), merge_first=1))
    b = gpu_decode(D, L, F.config(3, theta=float("inf")))
    assert (a["scores"] != b["scores"]).any()  # merged groups carry more mass than lone members
    wl, D, L, _, _ = synth.workload_inputs("c4", B=2)
    with pytest.raises(F.FlexCTCError):
        F.decode_nbest(torch.from_numpy(D).cuda(), torch.from_numpy(L).cuda(), wl_cfg(wl, merge_first=1), 2,
                       lm_pair[0], bt_pair[0])


def test_host_entry(lm_pair, bt_pair):
    """flexctc_decode_host (streamed H2D, the kernel polls the landed frames) with the variant."""
    wl, D, L, _, _ = synth.workload_inputs("c4", B=5)
    cfg = wl_cfg(wl, merge_first=1)
    ref = gpu_decode(D, L, cfg, lm_pair[0], bt_pair[0], alignment=False)
    out = F.decode_host(np.ascontiguousarray(D), np.asarray(L, np.int32), cfg, lm_pair[0], bt_pair[0])
    assert np.array_equal(out["num_tokens"], ref["num_tokens"])
    assert np.array_equal(out["tokens"], ref["tokens"])
    assert np.array_equal(np.asarray(out["scores"]).view(np.int32), ref["scores"].view(np.int32))
