"""GPU parity, round 2: the hand fixtures of tests/golden (timestamps R20, TopK tie SPEC S:342,
merge tie SPEC S:98) through both beam kernels, full-c5 parity in both combiners, and parity at
the batch sizes where the launch policy selects the 64-thread CTA variant (148 < B <= 592) and
the warp-per-utterance kernel (B > 592). Tokens, timestamps and alignments identical; scores
within 1e-4 (bit-identical in max mode)."""
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
from tests.test_gpu_parity import gpu_decode, run_pair, wl_cfg  # noqa: E402


def _path(monkeypatch, warp):
    """"0": the persistent CTA kernel, "1": the warp kernel."""
    monkeypatch.setenv("FLEXCTC_WARP", warp)


def _peaky(align, Vp1, p):
    D = np.full((len(align), Vp1), (1.0 - p) / (Vp1 - 1))
    D[np.arange(len(align)), align] = p
    return np.log(D)


@pytest.mark.parametrize("warp", ["0", "1"])
@pytest.mark.parametrize("mode", [0, 1])
def test_timestamp_fixtures(golden, monkeypatch, warp, mode):
    _path(monkeypatch, warp)
    g = golden["decode"]["timestamps"]
    for case in g["cases"]:
        D = _peaky(case["align"], 3, g["p_target"]).astype(np.float32)[None]
        out = gpu_decode(D, [len(case["align"])], F.config(4, theta=float("inf"), merge_mode=mode))
        n = int(out["num_tokens"][0])
        assert out["tokens"][0, :n].tolist() == case["tokens"]
        assert out["timestamps"][0, :n].tolist() == case["timestamps"]
        assert out["alignment"][0].tolist() == case["align"]


@pytest.mark.parametrize("warp", ["0", "1"])
def test_topk_tie_fixture(golden, monkeypatch, warp):
    _path(monkeypatch, warp)
    g = golden["decode"]["topk_tie"]
    D = np.log(np.array(g["D"], dtype=np.float64)).astype(np.float32)[None]
    out = gpu_decode(D, [1], F.config(g["beam"], theta=float("inf")))
    assert out["tokens"][0, :int(out["num_tokens"][0])].tolist() == g["nbest_tokens"][0]
    if warp == "0":  # n-best runs on the CTA kernel: both tied hypotheses, in slot order
        nb = F.decode_nbest(torch.from_numpy(D).cuda(), torch.tensor([1], dtype=torch.int32).cuda(),
                            F.config(g["beam"], theta=float("inf")), 2)
        torch.cuda.synchronize()
        got = [nb["tokens"][0, r, :int(nb["num_tokens"][0, r])].tolist() for r in range(2)]
        assert got == g["nbest_tokens"]
        assert float(nb["scores"][0, 0]) == float(nb["scores"][0, 1])


@pytest.mark.parametrize("warp", ["0", "1"])
@pytest.mark.parametrize("mode", [0, 1])
def test_merge_tie_fixture(golden, monkeypatch, warp, mode):
    _path(monkeypatch, warp)
    g = golden["decode"]["merge_tie"]
    D = np.log(np.array(g["D"], dtype=np.float64)).astype(np.float32)[None]
    out = gpu_decode(D, [2], F.config(g["beam"], theta=float("inf"), merge_mode=mode))
    assert out["tokens"][0, :int(out["num_tokens"][0])].tolist() == g["tokens"]
    assert out["timestamps"][0, :1].tolist() == g["timestamps"]
    assert out["alignment"][0].tolist() == g["alignment"]
    want = math.log(0.5) + math.log(0.7) if mode == 1 else math.log(0.85)
    assert float(out["scores"][0]) == pytest.approx(want, abs=1e-6)


@pytest.mark.parametrize("mode", [0, 1])
def test_c5_full(lm_pair, bt_pair, mode):
    """BASELINE configs[4] (B=512 LibriSpeech-shaped, K=128, LM + 1000 phrases), every utterance,
    log-sum-exp and max merges."""
    wl, D, L, _, _ = synth.workload_inputs("c5")
    run_pair(D, L, wl_cfg(wl, merge_mode=mode), lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1], ctx=f"c5 m{mode}")


@pytest.mark.parametrize("B", [400, 600])
def test_c4_shaped_large_batches(lm_pair, bt_pair, B):
    """c4-shaped batches where the launch policy picks the 64-thread CTA variant
    <64, 2, false, 1025, 16, 16, 7> (B = 400) and the warp-per-utterance kernel (B = 600 > 4 x 148)."""
    wl, D, L, _, _ = synth.workload_inputs("c4", B=B)
    run_pair(D, L, wl_cfg(wl), lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1], ctx=f"c4 B={B}")


@pytest.mark.parametrize("wname", ["c2", "c3", "c4"])
@pytest.mark.parametrize("mode", [0, 1])
def test_warp_kernel_forced(lm_pair, bt_pair, monkeypatch, wname, mode):
    """The warp kernel (and its compaction pass) at the small-batch configurations."""
    monkeypatch.setenv("FLEXCTC_WARP", "1")
    wl, D, L, _, _ = synth.workload_inputs(wname)
    glm, olm = (lm_pair[0], lm_pair[1]) if wl.lm else (None, None)
    gbt, obt = (bt_pair[0], bt_pair[1]) if wl.boost else (None, None)
    run_pair(D, L, wl_cfg(wl, merge_mode=mode), glm, olm, gbt, obt, ctx=f"warp {wname} m{mode}")


@pytest.mark.parametrize("cmp", ["0", "1"])
@pytest.mark.parametrize("wname", ["c3", "c4"])
@pytest.mark.parametrize("mode", [0, 1])
def test_cta_kernel_with_compaction_records(lm_pair, bt_pair, monkeypatch, wname, mode, cmp):
    """The persistent CTA kernel with (FLEXCTC_CMP=1: each frame's best token, listed band and
    floor from the compaction pass's records; the default for the c4 shape) and without
    (FLEXCTC_CMP=0: its own per-frame summaries) the records; both with the settled-beam fast path,
    and once without it."""
    monkeypatch.setenv("FLEXCTC_WARP", "0")
    monkeypatch.setenv("FLEXCTC_CMP", cmp)
    wl, D, L, _, _ = synth.workload_inputs(wname)
    glm, olm = (lm_pair[0], lm_pair[1]) if wl.lm else (None, None)
    gbt, obt = (bt_pair[0], bt_pair[1]) if wl.boost else (None, None)
    run_pair(D, L, wl_cfg(wl, merge_mode=mode), glm, olm, gbt, obt, ctx=f"records {wname} m{mode}")


def test_cta_kernel_without_fast_path(lm_pair, bt_pair, monkeypatch):
    """FLEXCTC_FAST=0: every frame through the general phases (the fast path's A/B switch)."""
    monkeypatch.setenv("FLEXCTC_FAST", "0")
    wl, D, L, _, _ = synth.workload_inputs("c4")
    run_pair(D, L, wl_cfg(wl), lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1], ctx="no fast path c4")


def test_cta_kernel_with_compaction_records_k128(lm_pair, bt_pair, monkeypatch):
    """The same at K = 128 (whole-CTA mode: the record's best token, the list instead of the row
    scan) on c5-shaped utterances."""
    monkeypatch.setenv("FLEXCTC_CMP", "1")
    wl, D, L, _, _ = synth.workload_inputs("c5", B=24)
    run_pair(D, L, wl_cfg(wl), lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1], ctx="records c5 B=24")


@pytest.mark.parametrize("rows", ["0", "4"])
def test_warp_kernel_row_cache_sizes(lm_pair, bt_pair, monkeypatch, rows):
    """The warp kernel with the dense-row cache off / tiny (evictions on every frame) at c4."""
    monkeypatch.setenv("FLEXCTC_WARP", "1")
    monkeypatch.setenv("FLEXCTC_WARP_ROWS", rows)
    wl, D, L, _, _ = synth.workload_inputs("c4", B=16)
    run_pair(D, L, wl_cfg(wl), lm_pair[0], lm_pair[1], bt_pair[0], bt_pair[1], ctx=f"rows {rows}")


def test_planted_spike_match_rate_c4(lm_pair, bt_pair):
    """R20 weak pin at c4 on the GPU path: decoded tokens sit at planted spike frames."""
    wl = synth.WORKLOADS["c4"]
    L = synth.lengths(wl, wl.B, wl.seed)
    D, tr, frames = synth.logprobs(wl.B, wl.T, wl.V, L, wl.seed, phrase_list=synth.phrases(wl.V), return_frames=True)
    g = gpu_decode(D, L, wl_cfg(wl), lm_pair[0], bt_pair[0])
    at = tot = 0
    for b in range(wl.B):
        n = int(g["num_tokens"][b])
        pl = set(frames[b])
        ts = g["timestamps"][b, :n].tolist()
        at += sum(int(x in pl) for x in ts)
        tot += n
    rate = at / tot
    print(f"c4 planted-spike timestamp match: {rate:.4f} of {tot} tokens")
    assert rate >= 0.95


@pytest.mark.parametrize("streamed", [True, False])
@pytest.mark.parametrize("wname,B", [("c4", 8), ("c5", 24), ("c1", 1)])
def test_decode_host_bf16(lm_pair, bt_pair, wname, B, streamed, monkeypatch):
    """flexctc_decode_host_bf16 (bf16 logits from the host, 2 B per logit over PCIe, normalised on
    the device chunk by chunk) == the oracle decoding the oracle's log-softmax of the same bits;
    and its device flags come back (0 here)."""
    from tests.test_gpu_logits import bf16_bits
    from tests.test_gpu_parity import compare, ocfg
    if not streamed:
        monkeypatch.setenv("FLEXCTC_NO_STREAM_INPUT", "1")
    wl, D, L, _, _ = synth.workload_inputs(wname, B=B)
    shift = np.random.default_rng(7).uniform(-5, 5, D.shape[:2] + (1,)).astype(np.float32)
    bits = np.ascontiguousarray(bf16_bits(D + shift))
    cfg = wl_cfg(wl, beam=min(wl.beam, 16))
    glm = lm_pair[0] if wl.lm else None
    gbt = bt_pair[0] if wl.boost else None
    xp = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).pin_memory()
    Lp = torch.from_numpy(L.astype(np.int32)).pin_memory()
    for _ in range(2):
        out = F.decode_host_bf16(xp, Lp, cfg, glm, gbt)
        assert out["flags"] == 0
        g = {k: (v.numpy() if hasattr(v, "numpy") else v) for k, v in out.items()}
        o = oracle.decode(oracle.log_softmax_bf16(bits), L, ocfg(cfg), lm_pair[1] if wl.lm else None,
                          bt_pair[1] if wl.boost else None)
        compare(g, o, ctx=f"host bf16 {wname}")


def test_decode_host_reports_length_flags():
    """decode_host returns the device flags: a length > T is clamped and flagged."""
    D = synth.random_logprobs(np.random.default_rng(3), 2, 6, 5, peak=4.0).astype(np.float32)
    out = F.decode_host(torch.from_numpy(D).pin_memory(), torch.tensor([9, 6], dtype=torch.int32).pin_memory(),
                        F.config(4))
    assert out["flags"] & F.flexctc.FLAG_LENGTH_CLAMPED_HIGH


def test_bindings_refuse_bad_lengths():
    """int64 / strided / wrong-size / wrong-device lengths raise instead of being misread."""
    D = torch.zeros((2, 4, 5), device="cuda")
    cfg = F.config(2)
    for bad in (torch.tensor([4, 3], dtype=torch.int64, device="cuda"),
                torch.tensor([4, 0, 3, 0], dtype=torch.int32, device="cuda")[::2],
                torch.tensor([4, 3, 2], dtype=torch.int32, device="cuda"),
                torch.tensor([4, 3], dtype=torch.int32)):
        for fn in (lambda L: F.decode(D, L, cfg), lambda L: F.decode_nbest(D, L, cfg, 2),
                   lambda L: F.decode_logits_bf16(D.to(torch.bfloat16), L, cfg)):
            with pytest.raises(F.FlexCTCError):
                fn(bad)


def _shard_worker(rank, ws, port, q):
    import os as _os
    import torch as _t
    import torch.distributed as dist
    _os.environ["MASTER_ADDR"] = "127.0.0.1"
    _os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import paper_2508_07315_b200 as F2
    import synth as S
    from paper_2508_07315_b200.shard import gather_results, lpt_assign
    from tests.test_gpu_parity import wl_cfg as wcfg
    _t.cuda.set_device(0)
    wl, D, L, arpa, ph = S.workload_inputs("c5")
    idx = lpt_assign(L, ws)[rank]
    lm, bt = F2.LM(arpa, wl.V, device=0), F2.Boost(ph, 1.0, wl.V, device=0)
    out = F2.decode(_t.from_numpy(np.ascontiguousarray(D[idx])).cuda(), _t.from_numpy(L[idx]).cuda(), wcfg(wl), lm, bt)
    _t.cuda.synchronize()
    g = gather_results({k: v.cpu() for k, v in out.items()}, idx, wl.B, D.shape[1], device=_t.device("cpu"))
    if rank == 0:
        q.put({k: v.numpy() for k, v in g.items()})
    dist.destroy_process_group()


def test_sharded_decode_matches_single_rank(lm_pair, bt_pair):
    """c5 LPT-sharded over 2 ranks (gloo, both on cuda:0) and gathered gives exactly
    the 1-rank decode of the whole batch, utterance by utterance."""
    import socket
    import torch.multiprocessing as mp
    wl, D, L, _, _ = synth.workload_inputs("c5")
    ref = gpu_decode(D, L, wl_cfg(wl), lm_pair[0], bt_pair[0], alignment=False)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert np.array_equal(got["num_tokens"], ref["num_tokens"])
    assert np.array_equal(got["tokens"], ref["tokens"])
    assert np.array_equal(got["timestamps"], ref["timestamps"])
    assert np.array_equal(got["scores"].view(np.int32), ref["scores"].view(np.int32))


@pytest.mark.parametrize("wname,B,K,mode", [("c4", 12, 16, 0), ("c4", 12, 16, 1), ("c3", 8, 16, 0), ("c5", 6, 128, 0),
                                            ("c4", 6, 1, 0), ("c4", 6, 4, 1)])
def test_fuse_repeats_variant(lm_pair, bt_pair, wname, B, K, mode):
    """the P:167 variant (LM / BT also on every repeated emission) on the GPU
    (the CTA kernel: K = 1 and the warp path route there) against the oracle's flag."""
    wl, D, L, _, _ = synth.workload_inputs(wname, B=B)
    glm, olm = (lm_pair[0], lm_pair[1]) if wl.lm else (None, None)
    gbt, obt = (bt_pair[0], bt_pair[1]) if wl.boost else (None, None)
    run_pair(D, L, wl_cfg(wl, beam=K, merge_mode=mode, fuse_repeats=1), glm, olm, gbt, obt,
             ctx=f"fuse_repeats {wname} K{K}")


def test_fuse_repeats_changes_scores(lm_pair, bt_pair):
    """The flag is live: on c4 utterances with repeated spikes the scores differ from Alg. 1."""
    wl, D, L, _, _ = synth.workload_inputs("c4", B=8)
    a = gpu_decode(D, L, wl_cfg(wl, fuse_repeats=1), lm_pair[0], bt_pair[0])
    b = gpu_decode(D, L, wl_cfg(wl), lm_pair[0], bt_pair[0])
    assert (a["scores"] != b["scores"]).any()
