"""GPU parity of flexctc_decode_logits_bf16 (log-softmax of bf16 logits on
the decoder's input side, reading R25) against the oracle decoding the oracle's own log-softmax
of the same bf16 logits."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2508_07315_b200 as F  # noqa: E402
import synth  # noqa: E402
from tests.test_gpu_parity import compare, ocfg, wl_cfg  # noqa: E402


def bf16_bits(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def gpu_logits(bits, L, cfg, lm=None, bt=None):
    x = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda().view(torch.bfloat16)
    out = F.decode_logits_bf16(x, torch.from_numpy(np.asarray(L, np.int32)).cuda(), cfg, lm, bt, alignment=True)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("wname,B,K", [("c1", None, 4), ("c2", 8, 8), ("c3", 8, 16), ("c4", 8, 16), ("c5", 12, 128),
                                       ("c4", 4, 1)])
def test_logits_bf16_vs_oracle(lm_pair, bt_pair, wname, B, K):
    wl, D, L, _, _ = synth.workload_inputs(wname, B=B)
    # logits: the synthetic log-probs shifted per frame (log-softmax is shift invariant) and
    # rounded to bf16 (coarse: many exact ties, which exercise the index tie rule R9)
    shift = np.random.default_rng(7).uniform(-5, 5, D.shape[:2] + (1,)).astype(np.float32)
    bits = bf16_bits(D + shift)
    Dq = oracle.log_softmax_bf16(bits)
    cfg = wl_cfg(wl, beam=K)
    glm = lm_pair[0] if wl.lm else None
    gbt = bt_pair[0] if wl.boost else None
    g = gpu_logits(bits, L, cfg, glm, gbt)
    o = oracle.decode(Dq, L, ocfg(cfg), lm_pair[1] if wl.lm else None, bt_pair[1] if wl.boost else None,
                      with_alignment=True)
    compare(g, o, ctx=f"logits {wname} K{K}")


def test_logits_bf16_strided_and_nan_padding():
    rng = np.random.default_rng(9)
    B, T, Vp1 = 5, 33, 129
    D = synth.random_logprobs(rng, B, T, Vp1, peak=5.0).astype(np.float32)
    bits = bf16_bits(D)
    padded = np.full((B, T, Vp1 + 3), 0x7FC0, np.uint16)  # bf16 NaN in the padding columns
    padded[:, :, :Vp1] = bits
    L = [33, 0, 1, 20, 32]
    for b, l in enumerate(L):
        padded[b, l:, :] = 0x7FC0  # frames t >= L_b are never read (R16)
    x = torch.from_numpy(padded.view(np.int16)).cuda().view(torch.bfloat16)[:, :, :Vp1]
    ws = F.flexctc.make_logits_workspace(B, T, Vp1, F.config(4))
    ws.buf.fill_(0xFF)  # NaN-filled workspace: rows t >= L_b of the normalised buffer are never read either
    out = F.decode_logits_bf16(x, torch.tensor(L, dtype=torch.int32, device="cuda"), F.config(4), workspace=ws,
                               alignment=True)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    Dq = oracle.log_softmax_bf16(bits)
    o = oracle.decode(Dq, L, ocfg(F.config(4)), with_alignment=True)
    compare(g, o)


@pytest.mark.parametrize("direct", ["1", "0"])
@pytest.mark.parametrize("mode", [0, 1])
def test_logits_direct_cta_path(lm_pair, bt_pair, monkeypatch, direct, mode):
    """The north-star shape at B <= #SMs: the CTA kernel stages the bf16 rows itself and normalises
    them with the compaction records' lse (FLEXCTC_LOGITS_DIRECT=1, the default) or decodes the
    dense fp32 copy of the normalisation pass (=0). Ragged lengths incl. 0 and 1, unaligned rows
    (V' = 1025 bf16 = 2050 B per row), the tensor's first and last rows at the buffer edges."""
    if direct == "0":
        monkeypatch.setenv("FLEXCTC_LOGITS_DIRECT", "0")
    wl, D, L, _, _ = synth.workload_inputs("c4", B=10)
    L = L.copy()
    L[1], L[4], L[7] = 0, 1, 217
    shift = np.random.default_rng(11).uniform(-5, 5, D.shape[:2] + (1,)).astype(np.float32)
    bits = bf16_bits(D + shift)
    Dq = oracle.log_softmax_bf16(bits)
    cfg = wl_cfg(wl, merge_mode=mode)
    g = gpu_logits(bits, L, cfg, lm_pair[0], bt_pair[0])
    o = oracle.decode(Dq, L, ocfg(cfg), lm_pair[1], bt_pair[1], with_alignment=True)
    compare(g, o, bitwise=mode == 1, ctx=f"logits direct={direct} mode={mode}")
    if mode == 0:  # the records path (lse only); with direct = 1 the kernel staged the bf16 rows itself
        assert F.flexctc.last_kernel() == ("ctc_beam_kernel+records+bf16" if direct == "1" else "ctc_beam_kernel+records")
