"""GPU parity of the greedy (beam K = 1) kernels, SURVEY §8(f) NEXT row 1 (PAPER Table II greedy
rows P:183-186; greedy + NGPU-LM P:80): the plain path (frame_top2_kernel + greedy_chain_kernel,
β = 0 without fusion) and the fused warp-per-utterance path (β, LM, boosting) against the oracle
at K = 1 and against the beam kernel at K = 1 (FLEXCTC_GREEDY=0), element by element."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2508_07315_b200 as F  # noqa: E402
import synth  # noqa: E402
from tests.test_gpu_parity import compare, gpu_decode, ocfg, run_pair, wl_cfg  # noqa: E402


def beam_kernel_k1(monkeypatch, D, L, cfg, lm=None, bt=None):
    monkeypatch.setenv("FLEXCTC_GREEDY", "0")
    try:
        return gpu_decode(D, L, cfg, lm, bt)
    finally:
        monkeypatch.delenv("FLEXCTC_GREEDY")


def same(a, b):
    for k in ("num_tokens", "tokens", "timestamps", "alignment"):
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(a["scores"].view(np.int32), b["scores"].view(np.int32))


def test_plain_greedy_c2_vs_oracle():
    """c2 shapes (B=32, T=400, V'=1025), β = 0, no fusion: the HBM-streaming path; bit-identical."""
    wl, D, L, _, _ = synth.workload_inputs("c2")
    run_pair(D, L, wl_cfg(wl, beam=1, merge_mode=1), bitwise=True, ctx="plain greedy c2")


@pytest.mark.parametrize("wname,lm,bt,beta", [("c2", False, False, 0.0), ("c2", False, False, 0.5),
                                                ("c3", True, False, 0.5), ("c4", True, True, 0.5),
                                                ("c4", True, True, -1.0), ("c5", True, True, 0.5)])
def test_greedy_kernels_equal_beam_kernel(lm_pair, bt_pair, monkeypatch, wname, lm, bt, beta):
    wl, D, L, _, _ = synth.workload_inputs(wname, B=48 if wname == "c5" else None)
    cfg = wl_cfg(wl, beam=1, beta=beta, alpha_lm=0.5 if lm else 0.0, alpha_bt=1.0 if bt else 0.0)
    glm, gbt = (lm_pair[0] if lm else None), (bt_pair[0] if bt else None)
    same(gpu_decode(D, L, cfg, glm, gbt), beam_kernel_k1(monkeypatch, D, L, cfg, glm, gbt))


def test_fused_greedy_negative_weights_and_retraction(lm_pair, bt_pair, monkeypatch):
    """α < 0 disables the bound (every token scored); EOS boost retraction (R17)."""
    wl, D, L, _, _ = synth.workload_inputs("c4", B=8)
    cfg = F.config(1, alpha_lm=-0.3, alpha_bt=1.0, beta=0.2, retract_boost_at_eos=1)
    run_pair(D, L, cfg, lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1], ctx="fused greedy alpha<0 retract")
    same(gpu_decode(D, L, cfg, lm_pair[0], bt_pair[0]), beam_kernel_k1(monkeypatch, D, L, cfg, lm_pair[0], bt_pair[0]))


def test_plain_greedy_rounding_tie():
    """A runner-up d2 < d1 at a lower index whose fl(acc + d2) equals fl(acc + d1): K = 1 of
    Alg. 1 takes the lower index (R9). The plain path must see it (rescan of that row)."""
    T, Vp1 = 400, 9
    D = np.full((2, T, Vp1), -10.0, np.float32)
    D[:, :, Vp1 - 1] = -2.5                    # blank dominates: acc reaches about -1000
    D[0, T - 1, 5] = -1.0
    D[0, T - 1, 2] = np.float32(-1.0) - np.float32(2e-5)  # ulp(1000) = 6.1e-5: ties after rounding
    D[1, T - 1, 5] = -1.0
    D[1, T - 1, 2] = -1.5                      # a clear winner: no tie
    L = [T, T]
    cfg = F.config(1, theta=12.0)
    g = gpu_decode(D, L, cfg)
    o = oracle.decode(D, L, ocfg(cfg), nthreads=1, with_alignment=True)
    compare(g, o, bitwise=True)
    assert g["tokens"][0, 0] == 2 and g["tokens"][1, 0] == 5
    assert g["alignment"][0, T - 1] == 2


def test_greedy_dead_zero_length_and_nan_padding(lm_pair, monkeypatch):
    Vp1 = 1025
    rng = np.random.default_rng(5)
    D = synth.random_logprobs(rng, 4, 30, Vp1, peak=6.0).astype(np.float32)
    D[1, 7, :] = -np.inf                       # no finite candidate: the hypothesis dies
    D[2, 12:, :] = np.nan                      # padding (L = 12) is never read
    L = [30, 30, 12, 0]
    for cfg, lm in ((F.config(1), None), (F.config(1, alpha_lm=0.5, beta=0.5), lm_pair)):
        g = gpu_decode(D, L, cfg, lm[0] if lm else None)
        o = oracle.decode(np.where(np.isnan(D), np.float32(-1.0), D), L, ocfg(cfg), lm[1] if lm else None, None, 1,
                          with_alignment=True)
        compare(g, o, bitwise=True)
        assert g["num_tokens"][1] == 0 and g["scores"][1] == -np.inf and g["num_tokens"][3] == 0
        same(g, beam_kernel_k1(monkeypatch, D, L, cfg, lm[0] if lm else None))


@pytest.mark.parametrize("pad", [0, 1, 3, 6])
def test_plain_greedy_strides(pad):
    """Row stride V' + pad (rows start at every 4-B phase): head / body / tail of the 16-B loads."""
    rng = np.random.default_rng(11 + pad)
    B, T, Vp1 = 5, 37, 129
    D = synth.random_logprobs(rng, B, T, Vp1, peak=4.0).astype(np.float32)
    Dp = np.full((B, T, Vp1 + pad), np.nan, np.float32)
    Dp[:, :, :Vp1] = D
    L = [37, 1, 20, 36, 0]
    g = gpu_decode(torch.from_numpy(Dp).cuda()[:, :, :Vp1], L, F.config(1))
    o = oracle.decode(D, L, ocfg(F.config(1)), nthreads=1, with_alignment=True)
    compare(g, o, bitwise=True)


def test_greedy_zero_frames(lm_pair):
    """T = 0 (every length 0): empty transcripts, score = α_LM·LM.Final(<s>) (reading of §8(b))."""
    D = np.zeros((3, 1, 1025), np.float32)  # the oracle's view: one frame, never read (L = 0)
    for cfg, lm in ((F.config(1), None), (F.config(1, alpha_lm=0.5, beta=0.5), lm_pair)):
        g = gpu_decode(torch.zeros((3, 0, 1025), device="cuda"), [0, 0, 0], cfg, lm[0] if lm else None)
        o = oracle.decode(D, [0, 0, 0], ocfg(cfg), lm[1] if lm else None, None, 1, with_alignment=True)
        assert g["tokens"].shape == (3, 0)
        assert g["num_tokens"].tolist() == [0, 0, 0] == o["num_tokens"].tolist()
        assert np.array_equal(g["scores"].view(np.int32), o["scores"].view(np.int32))


@pytest.mark.parametrize("Vp1", [4097, 5000, 8192])
def test_large_vocab_greedy_and_beam(Vp1):
    """V' beyond one 16-B-load batch per lane (frame_summary_kernel folds the arg-max across
    batches) and up to the 8192 limit; the fused path and the beam kernel at the same size."""
    rng = np.random.default_rng(Vp1)
    B, T = 3, 24
    D = synth.random_logprobs(rng, B, T, Vp1, peak=8.0).astype(np.float32)
    D[0, 5, 4100:4110] = D[0, 5].max()  # exact ties of the max in the second batch region
    D[1, 7, [3, Vp1 - 40]] = D[1, 7].max() + 1.0  # the max in the first and the second batch
    L = [24, 24, 9]
    for cfg in (F.config(1), F.config(1, beta=0.3), F.config(4, theta=12.0)):
        g = gpu_decode(D, L, cfg)
        o = oracle.decode(D, L, ocfg(cfg), nthreads=1, with_alignment=True)
        compare(g, o, bitwise=cfg.beam == 1)
