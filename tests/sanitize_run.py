"""Small decodes for compute-sanitizer (memcheck / racecheck / synccheck), SURVEY.md §4 item 5.

  compute-sanitizer --tool racecheck python tests/sanitize_run.py

Covers the beam-warp + helpers mode (K <= 32, LM + boosting), the whole-CTA mode (K = 64), the
single-warp launch, the greedy kernels (plain and fused, K = 1; TMA bulk rows + mbarriers), the
n-best output, the bf16-logits input pass and the streamed host path, on a few short utterances,
and checks the results against the oracle. Round 2: the compaction pass (TMA-staged), the warp
kernel, the CTA kernel reading compaction records, and the merge-before-TopK kernel."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2508_07315_b200 as F  # noqa: E402
import synth  # noqa: E402


def run(K, nt=None):
    if nt:
        os.environ["FLEXCTC_NT"] = str(nt)
    else:
        os.environ.pop("FLEXCTC_NT", None)
    wl = synth.WORKLOADS["c4"]
    L = np.array([40, 17, 0], dtype=np.int32)
    ph = synth.phrases(1024)
    D, _ = synth.logprobs(3, 40, 1024, L, 5, ph)
    arpa = synth.arpa_file(V=1024)
    glm, gbt = F.LM(arpa, 1024, device=0), F.Boost(ph, 1.0, 1024, device=0)
    cfg = F.config(K, 0.5, 1.0, 0.5, 12.0)
    out = F.decode(torch.from_numpy(D).cuda(), torch.from_numpy(L).cuda(), cfg, glm, gbt)
    torch.cuda.synchronize()
    ref = oracle.decode(D, L, oracle.make_cfg(K, 0.5, 1.0, 0.5, 12.0), oracle.LM(arpa, 1024),
                        oracle.Boost(ph, 1.0, 1024), nthreads=4)
    assert np.array_equal(out["tokens"].cpu().numpy(), ref["tokens"]), K
    assert np.allclose(out["scores"].cpu().numpy(), ref["scores"], atol=1e-4), K
    print(f"K={K} nt={nt or 'default'} ok")


def run_more():
    os.environ.pop("FLEXCTC_NT", None)
    L = np.array([40, 17, 0, 33], dtype=np.int32)
    ph = synth.phrases(1024)
    D, _ = synth.logprobs(4, 40, 1024, L, 5, ph)
    arpa = synth.arpa_file(V=1024)
    glm, gbt = F.LM(arpa, 1024, device=0), F.Boost(ph, 1.0, 1024, device=0)
    olm, obt = oracle.LM(arpa, 1024), oracle.Boost(ph, 1.0, 1024)
    Dt, Lt = torch.from_numpy(D).cuda(), torch.from_numpy(L).cuda()

    def check(out, ref, what):
        assert np.array_equal(out["tokens"].cpu().numpy(), ref["tokens"]), what
        assert np.allclose(out["scores"].cpu().numpy(), ref["scores"], atol=1e-4), what
        print(what, "ok")

    for cfg, lm, bt in ((F.config(1), None, None), (F.config(1, 0.5, 1.0, 0.5, 12.0), glm, gbt)):
        out = F.decode(Dt, Lt, cfg, lm, bt)
        torch.cuda.synchronize()
        ref = oracle.decode(D, L, oracle.make_cfg(1, cfg.alpha_lm, cfg.alpha_bt, cfg.beta, 12.0),
                            olm if lm else None, obt if bt else None, nthreads=4)
        check(out, ref, f"greedy lm={lm is not None}")
    cfg = F.config(16, 0.5, 1.0, 0.5, 12.0)
    ref = oracle.decode(D, L, oracle.make_cfg(16, 0.5, 1.0, 0.5, 12.0), olm, obt, nthreads=4)
    nb = F.decode_nbest(Dt, Lt, cfg, 4, glm, gbt)
    torch.cuda.synchronize()
    check({"tokens": nb["tokens"][:, 0], "scores": nb["scores"][:, 0]}, ref, "nbest")
    hout = F.decode_host(torch.from_numpy(D).pin_memory(), torch.from_numpy(L).pin_memory(), cfg, glm, gbt)
    check(hout, ref, "decode_host streamed")
    u = D.view(np.uint32).astype(np.uint64)
    bits = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    Dq = oracle.log_softmax_bf16(bits)
    x = torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)
    for K in (16, 1):
        out = F.decode_logits_bf16(x, Lt, F.config(K, 0.5, 1.0, 0.5, 12.0), glm, gbt)
        torch.cuda.synchronize()
        check(out, oracle.decode(Dq, L, oracle.make_cfg(K, 0.5, 1.0, 0.5, 12.0), olm, obt, nthreads=4),
              f"logits bf16 K={K}")


def run_round2():
    """Round 2 kernels: the compaction pass + warp kernel (TMA rings, dense-row cache with
    evictions, boost signatures), the CTA kernel reading compaction records (K = 16 beam-warp mode
    and K = 64 whole-CTA mode)."""
    for env, K in ((dict(FLEXCTC_WARP="1"), 16), (dict(FLEXCTC_WARP="1", FLEXCTC_WARP_ROWS="2"), 16),
                   (dict(FLEXCTC_WARP="0", FLEXCTC_CMP="1"), 16), (dict(FLEXCTC_CMP="1"), 64)):
        os.environ.update(env)
        try:
            run(K)
        finally:
            for k in env:
                os.environ.pop(k, None)
        print("  with", env)


def run_merge_first():
    """merge_first_kernel (reading R27): the buffer cut (θ = ∞, K = 4 on flat V' = 9 frames forces
    repeated sorts) and the c4-shaped LM + boosting case."""
    rng = np.random.default_rng(2)
    D = synth.random_logprobs(rng, 3, 40, 9, peak=0.5).astype(np.float32)
    L = np.array([40, 13, 0], dtype=np.int32)
    out = F.decode(torch.from_numpy(D).cuda(), torch.from_numpy(L).cuda(), F.config(4, theta=float("inf"), merge_first=1))
    torch.cuda.synchronize()
    ref = oracle.decode(D, L, oracle.make_cfg(4, merge_first=1), nthreads=4)
    assert np.array_equal(out["tokens"].cpu().numpy(), ref["tokens"])
    assert np.allclose(out["scores"].cpu().numpy(), ref["scores"], atol=1e-4)
    L = np.array([40, 17, 0], dtype=np.int32)
    ph = synth.phrases(1024)
    D, _ = synth.logprobs(3, 40, 1024, L, 5, ph)
    arpa = synth.arpa_file(V=1024)
    glm, gbt = F.LM(arpa, 1024, device=0), F.Boost(ph, 1.0, 1024, device=0)
    out = F.decode(torch.from_numpy(D).cuda(), torch.from_numpy(L).cuda(), F.config(16, 0.5, 1.0, 0.5, 12.0, merge_first=1),
                   glm, gbt)
    torch.cuda.synchronize()
    ref = oracle.decode(D, L, oracle.make_cfg(16, 0.5, 1.0, 0.5, 12.0, merge_first=1), oracle.LM(arpa, 1024),
                        oracle.Boost(ph, 1.0, 1024), nthreads=4)
    assert np.array_equal(out["tokens"].cpu().numpy(), ref["tokens"])
    assert np.allclose(out["scores"].cpu().numpy(), ref["scores"], atol=1e-4)
    print("merge_first ok")


if __name__ == "__main__":
    run(16)
    run(64)
    run(16, nt=32)
    run_more()
    run_round2()
    run_merge_first()
