"""Debug helper (not collected by pytest): decode a workload on the GPU under the current env
and report utterances that differ from the oracle.  python tests/debug_compare.py c3 [B]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2508_07315_b200 as F  # noqa: E402
import synth  # noqa: E402


def main():
    name = sys.argv[1]
    B = int(sys.argv[2]) if len(sys.argv) > 2 else None
    mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    wl, D, L, arpa, ph = synth.workload_inputs(name, B=B)
    glm = F.LM(arpa, wl.V, device=0) if wl.lm else None
    gbt = F.Boost(ph, 1.0, wl.V, device=0) if wl.boost else None
    olm = oracle.LM(arpa, wl.V) if wl.lm else None
    obt = oracle.Boost(ph, 1.0, wl.V) if wl.boost else None
    cfg = F.config(wl.beam, wl.alpha_lm if wl.lm else 0, wl.alpha_bt if wl.boost else 0, wl.beta, wl.theta, mode)
    out = F.decode(torch.from_numpy(D).cuda(), torch.from_numpy(L).cuda(), cfg, glm, gbt, alignment=True)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    o = oracle.decode(D, L, oracle.make_cfg(wl.beam, cfg.alpha_lm, cfg.alpha_bt, wl.beta, wl.theta, mode), olm, obt,
                      with_alignment=True)
    bad = 0
    for b in range(D.shape[0]):
        same_tok = np.array_equal(g["tokens"][b], o["tokens"][b])
        same_al = np.array_equal(g["alignment"][b], o["alignment"][b])
        ds = float(g["scores"][b]) - float(o["scores"][b])
        if not same_tok or not same_al or abs(ds) > 1e-6:
            bad += 1
            fa = np.nonzero(g["alignment"][b] != o["alignment"][b])[0]
            print(f"utt {b}: tokens_equal={same_tok} align_equal={same_al} dscore={ds:.3e} "
                  f"first_align_diff={fa[:5].tolist()} gpu={g['scores'][b]} orc={o['scores'][b]}")
    print(f"{name}: {bad} of {D.shape[0]} utterances differ (env FLEXCTC_SOLO={os.environ.get('FLEXCTC_SOLO')})")


if __name__ == "__main__":
    main()
