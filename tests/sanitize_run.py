"""Small decodes for compute-sanitizer (memcheck / racecheck / synccheck), SURVEY.md §4 item 5.

  compute-sanitizer --tool racecheck python tests/sanitize_run.py

Covers the beam-warp + helpers mode (K <= 32, LM + boosting), the whole-CTA mode (K = 64) and the
single-warp launch, on a few short utterances, and checks the results against the oracle."""
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


if __name__ == "__main__":
    run(16)
    run(64)
    run(16, nt=32)
