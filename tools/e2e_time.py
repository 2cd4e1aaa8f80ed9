import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2508_07315_b200 as F, synth
for wname in ("c4", "c5"):
    wl, D, L, arpa, ph = synth.workload_inputs(wname)
    lm = F.LM(arpa, wl.V); bt = F.Boost(ph, 1.0, wl.V)
    cfg = F.config(wl.beam, wl.alpha_lm, wl.alpha_bt, wl.beta, wl.theta, wl.merge_mode)
    Dp = torch.from_numpy(D).pin_memory(); Lp = torch.from_numpy(L).pin_memory()
    B, T, Vp1 = D.shape
    scratch = torch.empty(F.host_scratch_bytes(B, T, Vp1, cfg), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    out = None
    for _ in range(3): out = F.decode_host(Dp, Lp, cfg, lm, bt, scratch=scratch, stream=s, out=out)
    ts = []; th = []
    for _ in range(10):
        t0 = time.perf_counter(); out = F.decode_host(Dp, Lp, cfg, lm, bt, scratch=scratch, stream=s, out=out); ts.append(time.perf_counter() - t0)
    print(wname, "e2e ms %.3f" % (1e3 * np.median(ts)), "streaming", F.host_streaming())
