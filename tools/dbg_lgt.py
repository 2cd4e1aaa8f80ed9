import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_07315_b200 as F, synth
from tests.test_gpu_logits import bf16_bits
wl, D, L, arpa, ph = synth.workload_inputs("c4", B=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
lm, bt = F.LM(arpa, 1024, device=0), F.Boost(ph, 1.0, 1024, device=0)
bits = bf16_bits(D)
x = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda().view(torch.bfloat16)
cfg = F.config(16, 0.5, 1.0, 0.5, 12.0)
out = F.decode_logits_bf16(x, torch.from_numpy(L).cuda(), cfg, lm, bt)
torch.cuda.synchronize()
print("ok", F.flexctc.last_kernel(), out["num_tokens"][:4].tolist())
