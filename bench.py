"""Benchmark of the FlexCTC hot path on B200 (driver contract).

One step = one flexctc_decode of the whole hot path (Alg. 1 over every frame of every
utterance of the rank's batch: frame read, candidates, LM/boost fusion, top-K, θ-prune, state
advance, recombination, EOS, backtrace) with inputs already resident in HBM. L2 is flushed
between steps (a 256 MiB write). Default workload: c4 = BASELINE.json configs[3] (B=64 per GPU,
T=400 @ 40 ms, V=1024+blank, beam 16, 4-gram LM, 1000 boosted phrases) — the configuration the
north-star metric is quoted on. Multi-GPU (torchrun): weak scaling, each rank decodes its own
c4 batch (distinct seeds), LM/boost replicated, results gathered once at the end.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4] [--impl flexctc|reference]
                  [--scaling weak|strong] [--stream M] [--input f32-logprobs|bf16-logits]

--gpus N without torchrun re-launches itself under torch.distributed.run with N ranks (one per
GPU, 127.0.0.1 rendezvous); under torchrun WORLD_SIZE must equal N. --scaling strong decodes ONE
global batch (the workload's batch, times --stream M) LPT-sharded over the ranks
(shard.lpt_assign) and reports each rank's share, critical path and the load balance.
"""
from __future__ import annotations

import argparse
import datetime
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "RTFx (audio s decoded / wall s) and frames·beams/s at 1/2/4/8 B200"
UNIT = "RTFx"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c4", choices=sorted(synth.WORKLOADS))
    ap.add_argument("--impl", default="flexctc", choices=["flexctc", "reference"])
    ap.add_argument("--batch", type=int, default=0, help="override the workload's batch per GPU")
    ap.add_argument("--input", default="f32-logprobs", choices=["f32-logprobs", "bf16-logits"],
                    help="bf16-logits: flexctc_decode_logits_bf16, log-softmax fused into the frame read (NEXT 4)")
    ap.add_argument("--beam", type=int, default=0,
                    help="override the workload's beam (1 = the greedy kernels, SURVEY §8(f) NEXT 1)")
    ap.add_argument("--merge-first", action="store_true",
                    help="the merge-before-TopK variant (config merge_first = 1, DESIGN.md reading R27)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="utterances in the oracle sample (0 = auto)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: each rank decodes its own batch; strong: one global batch LPT-sharded over the ranks")
    ap.add_argument("--stream", type=int, default=1,
                    help="strong scaling: the global batch is M x the workload batch (distinct seeds), e.g. 8 x 512")
    return ap.parse_args()


def spawn_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run with N ranks."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_config(wl, B, T, Lsum, extra=None):
    cfg = {"workload": wl.name, "B_per_gpu": B, "T": T, "V": wl.V, "beam": wl.beam,
           "lm": "synthetic 4-gram ARPA (~1.08M n-grams)" if wl.lm else None,
           "phrases": 1000 if wl.boost else 0, "alpha_lm": wl.alpha_lm if wl.lm else 0.0,
           "alpha_bt": wl.alpha_bt if wl.boost else 0.0, "beta": wl.beta, "theta": wl.theta,
           "merge": "lse" if wl.merge_mode == 0 else "max", "frame_s": synth.FRAME_SECONDS,
           "frames_per_gpu": int(Lsum), "l2": "flushed (256 MiB write) between timed steps"}
    if extra:
        cfg.update(extra)
    return cfg


class ClockSampler:
    """nvidia-smi clocks / throttle reasons; only samples whose nvidia-smi timestamp falls inside
    the timed region [mark_start(), mark_end()] are reported."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def mark_start(self):
        self.t0 = datetime.datetime.now()

    def mark_end(self):
        self.t1 = datetime.datetime.now()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)  # let the sampler emit the samples that cover the end of the region
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.th.join(timeout=2)
        inside = []
        for r in self.rows:
            if len(r) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f")
            except ValueError:
                continue
            if self.t0 and self.t1 and self.t0 <= ts <= self.t1 + datetime.timedelta(milliseconds=20):
                inside.append(r)
        sm = [float(r[1]) for r in inside if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in inside if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in inside:
            for n, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "region_ms": (self.t1 - self.t0).total_seconds() * 1e3 if self.t0 and self.t1 else None}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    e = d.get(workload)
    if not e:
        return None, None
    return e.get("dram_bytes_per_launch"), e.get("source")


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.TimeoutExpired):
        pass
    return "unknown"


def one_thread_times():
    """The oracle on ONE host thread over the whole c1 and c2 batches."""
    import oracle
    res = {}
    for name in ("c1", "c2"):
        wl, D, L, _, _ = synth.workload_inputs(name)
        cfg = oracle.make_cfg(wl.beam, 0.0, 0.0, wl.beta, wl.theta, wl.merge_mode)
        t0 = time.perf_counter()
        oracle.decode(D, L, cfg, nthreads=1)
        dt = time.perf_counter() - t0
        res[name] = {"s": round(dt, 4), "rtfx": float(L.sum()) * synth.FRAME_SECONDS / dt}
    return res


def cpu_baseline(wl, D, L, arpa, ph, n_utts, merge_first=0):
    """The oracle as it stands (never tuned), on this host's cores, over a bounded sample."""
    import oracle
    lm = oracle.LM(arpa, wl.V) if wl.lm else None
    bt = oracle.Boost(ph, 1.0, wl.V) if wl.boost else None
    cfg = oracle.make_cfg(wl.beam, wl.alpha_lm if wl.lm else 0.0, wl.alpha_bt if wl.boost else 0.0, wl.beta,
                          wl.theta, wl.merge_mode, merge_first=merge_first)
    cores = os.cpu_count() or 1
    idx = np.arange(min(n_utts, D.shape[0]))
    Ds = np.ascontiguousarray(D[idx])
    t0 = time.perf_counter()
    oracle.decode(Ds, L[idx], cfg, lm, bt, nthreads=cores)
    dt = time.perf_counter() - t0
    audio = float(L[idx].sum()) * synth.FRAME_SECONDS
    return {"value": audio / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{len(idx)} of the {wl.name} utterances ({int(L[idx].sum())} frames, "
                      f"{audio:.1f} audio s) decoded by the C++ oracle on {cores} host threads in {dt:.1f} s",
            "frames_beams_per_s": float(L[idx].sum()) * wl.beam / dt,
            "cpu_model": cpu_model(), "one_thread": one_thread_times()}


def run_reference(args):
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return
    wl = synth.WORKLOADS[args.workload]
    _, D, L, arpa, ph = synth.workload_inputs(args.workload)
    import oracle
    lm = oracle.LM(arpa, wl.V) if wl.lm else None
    bt = oracle.Boost(ph, 1.0, wl.V) if wl.boost else None
    cfg = oracle.make_cfg(wl.beam, wl.alpha_lm if wl.lm else 0.0, wl.alpha_bt if wl.boost else 0.0, wl.beta,
                          wl.theta, wl.merge_mode)
    cores = os.cpu_count() or 1
    # per step: 16 utterances (~0.3 s on 16 threads at c4) so that K steps stay within minutes
    n = args.cpu_sample or (min(wl.B, 16) if wl.beam <= 32 else min(wl.B, 4))
    idx = np.arange(n)
    Ds = np.ascontiguousarray(D[idx])
    for _ in range(args.warmup):
        oracle.decode(Ds, L[idx], cfg, lm, bt, nthreads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.decode(Ds, L[idx], cfg, lm, bt, nthreads=cores)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    frames = float(L[idx].sum())
    value = frames * synth.FRAME_SECONDS * args.steps / tot
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": workload_config(wl, int(n), int(D.shape[1]), L[idx].sum(),
                                     {"reference": "C++ oracle (oracle/oracle.cpp), host cores"}),
           "frames_beams_per_s": frames * wl.beam * args.steps / tot,
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": f"{n} utterances of {wl.name} per step on {cores} host threads"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_flexctc(args):
    import torch
    import torch.distributed as dist

    import paper_2508_07315_b200 as F
    from paper_2508_07315_b200 import flexctc as FX
    from paper_2508_07315_b200.shard import gather_results

    rank, world, local = dist_env()
    gpu = local % max(1, torch.cuda.device_count())  # ranks > GPUs only in the 1-GPU path test
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        backend = os.environ.get("FLEXCTC_DIST_BACKEND", "nccl")  # gloo: multi-rank test on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    wl = synth.WORKLOADS[args.workload]
    if args.beam:
        wl = dataclasses.replace(wl, beam=args.beam, name=f"{wl.name} (beam {args.beam})")
    strong = args.scaling == "strong"
    shard_idx = None
    if not strong:
        # weak scaling: rank r decodes its own batch of the workload (seed offset r)
        _, D, L, arpa, ph = synth.workload_inputs(args.workload, B=args.batch or None, seed_offset=rank)
    else:
        # strong scaling: one global batch (M x the workload batch, chunk m with seed offset m),
        # LPT-sharded by length over the ranks; each rank generates only its own rows
        from paper_2508_07315_b200.shard import lpt_assign
        Bw = args.batch or wl.B
        Ls = [synth.lengths(wl, Bw, wl.seed + m) for m in range(args.stream)]
        L_all = np.concatenate(Ls)
        shard_idx = lpt_assign(L_all, world)[rank]
        Tg = int(L_all.max()) if wl.lengths != "fixed" else wl.T
        mine = set(int(i) for i in shard_idx)
        D = np.zeros((len(shard_idx), Tg, wl.V + 1), dtype=np.float32)
        row = {int(g): j for j, g in enumerate(shard_idx)}
        arpa = ph = None
        for m in range(args.stream):
            lo = m * Bw
            if not any(lo <= i < lo + Bw for i in mine):
                continue
            _, Dm, Lm, arpa, ph = synth.workload_inputs(args.workload, B=Bw, seed_offset=m)
            for i in range(lo, lo + Bw):
                if i in mine:
                    D[row[i], :Dm.shape[1]] = Dm[i - lo]
            del Dm
        if arpa is None and wl.lm:
            arpa = synth.arpa_file(V=wl.V)
        if ph is None and wl.boost:
            ph = synth.phrases(wl.V)
        L = L_all[shard_idx].astype(np.int32)
    B, T, Vp1 = D.shape
    lm = F.LM(arpa, wl.V, device=gpu) if wl.lm else None
    bt = F.Boost(ph, 1.0, wl.V, device=gpu) if wl.boost else None
    cfg = F.config(wl.beam, wl.alpha_lm if wl.lm else 0.0, wl.alpha_bt if wl.boost else 0.0, wl.beta, wl.theta,
                   wl.merge_mode, merge_first=int(args.merge_first))
    Dd = torch.from_numpy(D).to(dev)
    bf16 = args.input == "bf16-logits"
    if bf16:  # the synthetic log-probs as bf16 logits (log-softmax is shift invariant)
        Dd = Dd.to(torch.bfloat16)
    Ld = torch.from_numpy(L).to(dev)
    ws = FX.make_logits_workspace(B, T, Vp1, cfg, dev) if args.input == "bf16-logits" else F.make_workspace(B, T, Vp1, cfg, dev)
    stream = torch.cuda.Stream(dev)
    out = None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # per step: decode start/stop, beam kernel start/stop (stage 0), compaction pass start/stop (stage 1)
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(6)) for _ in range(args.steps)]
    for e in ev:  # torch creates events lazily: record once so the C hook gets real cudaEvent_t handles
        for x in e[2:]:
            x.record(stream)

    def step(e=None):
        nonlocal out
        with torch.cuda.stream(stream):
            flush.fill_(1)  # evict L2 (126 MB) between steps; not timed
            if e is not None:
                e[0].record(stream)
                FX.set_stage_events(0, e[2], e[3])
                FX.set_stage_events(1, e[4], e[5])
            if bf16:
                out = F.decode_logits_bf16(Dd, Ld, cfg, lm, bt, workspace=ws, stream=stream, outputs=out)
            else:
                out = F.decode(Dd, Ld, cfg, lm, bt, workspace=ws, stream=stream, outputs=out)
            if e is not None:
                e[1].record(stream)
                FX.set_stage_events(0, None, None)
                FX.set_stage_events(1, None, None)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    kernel_name = FX.last_kernel()
    compacted = kernel_name.startswith("warp_beam_kernel")  # the warp path runs the compaction pass
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(gpu)
    clocks.start()
    time.sleep(0.15)  # let nvidia-smi start sampling before the timed region opens
    clocks.mark_start()
    for i in range(args.steps):
        step(ev[i])
    torch.cuda.synchronize()
    clocks.mark_end()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_dec = sum(e[0].elapsed_time(e[1]) for e in ev) / 1e3        # s, whole decode per step summed
    t_kern = sum(e[2].elapsed_time(e[3]) for e in ev) / 1e3       # s, beam kernel only
    compacted = compacted or "+records" in kernel_name  # CTA kernel reading the records
    t_cmp = sum(e[4].elapsed_time(e[5]) for e in ev) / 1e3 if compacted else 0.0  # s, compaction pass
    t_dec_local = t_dec
    flags = F.check(ws)
    dstats = FX.stats(ws)  # device counters of the last timed decode
    tt = torch.tensor([t_dec, t_kern, t_cmp], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_dec, t_kern, t_cmp = float(tt[0]), float(tt[1]), float(tt[2])
    frames_local = float(L.sum())
    frames_all = frames_local * world  # weak scaling: same frame count per rank (c4: fixed T)
    if world > 1:
        fa = torch.tensor([frames_local], dtype=torch.float64, device=dev)
        dist.all_reduce(fa)
        frames_all = float(fa[0])
    value = frames_all * synth.FRAME_SECONDS * args.steps / t_dec
    fbps = frames_all * wl.beam * args.steps / t_dec
    shards = None
    if strong:  # each rank's share and critical path (LPT balance)
        mine_t = torch.tensor([float(B), frames_local, float(L.max() if len(L) else 0),
                               1e3 * t_dec_local / args.steps], dtype=torch.float64, device=dev)
        allt = [torch.zeros_like(mine_t) for _ in range(world)]
        if world > 1:
            dist.all_gather(allt, mine_t)
        else:
            allt = [mine_t]
        shards = [{"rank": r, "utterances": int(x[0]), "frames": int(x[1]), "T_max": int(x[2]),
                   "ms_per_step": round(float(x[3]), 4)} for r, x in enumerate(allt)]
        fr = [sh["frames"] for sh in shards]

    # roofline of the dominant kernel: algorithmic bytes per launch =
    #  beam kernel:         Σ_b L_b · (4·V' [read D once] + 3·K [u8 parent + u16 label backpointers])
    #  plain greedy (K=1):  frame_top2_kernel, Σ_b L_b · (4·V' + 16 [{d1, w1, d2} frame summary])
    #  fused greedy (K=1):  greedy_fused_kernel, Σ_b L_b · 4·V'
    #  warp path (2 <= K <= 32): warp_beam_kernel reads each frame's row (4·V', or 2·V' bf16 logits)
    #                       and its 256-B record, writes 3·K B of backpointers; the compaction pass
    #                       reads the row and writes the record: Σ_b L_b · (4·V' + 256) (its own entry)
    plain_greedy = wl.beam == 1 and not wl.lm and not wl.boost and wl.beta == 0.0
    # bf16 logits: the compaction pass reads the logits (2 B) on the warp path and on the CTA path
    # that reads them directly (kernel "...+records+bf16"); elsewhere the CTA path normalises them
    # first into a dense fp32 buffer that the pass then reads (4 B)
    xb = 2 if bf16 and (kernel_name.startswith("warp_beam_kernel") or kernel_name.endswith("+bf16")) else 4
    roof_cmp = None
    if wl.beam > 1 and compacted:
        alg_bytes = frames_local * (xb * Vp1 + 256 + 3 * wl.beam)
        kname = kernel_name + " (beam warp per utterance" + (" + helper warps)" if "helpers" in kernel_name else ")")
        note = ("latency-bound recurrence: T_max dependent frame steps; the HBM stream of D is the "
                "compaction pass (roofline_compact); see DESIGN.md")
        cmp_bytes = frames_local * (xb * Vp1 + 256)
    elif wl.beam > 1:
        alg_bytes, kname = frames_local * (4 * Vp1 + 3 * wl.beam), "ctc_beam_kernel (persistent)"
        note = "latency-bound recurrence: T_max dependent frame steps; see DESIGN.md"
    elif plain_greedy:
        alg_bytes, kname = frames_local * (4 * Vp1 + 16), "frame_summary_kernel (HBM stream of D)"
        note = "fully parallel over frames: bandwidth-bound; see DESIGN.md"
    else:
        alg_bytes, kname = frames_local * 4 * Vp1, "greedy_fused_kernel (warp per utterance)"
        note = "latency-bound recurrence over T frames per utterance; see DESIGN.md"
    kern_s = t_kern / args.steps
    achieved = alg_bytes / kern_s / 1e9
    peak, peak_src = peaks()
    tkey = (args.workload if not args.beam else f"{args.workload}_k{args.beam}") + ("_bf16" if bf16 else "")
    traffic, traffic_src = ncu_traffic(tkey)
    if wl.beam > 1 and compacted and t_cmp > 0:
        cmp_s = t_cmp / args.steps
        ctraffic, ctraffic_src = ncu_traffic(tkey + "_compact")
        roof_cmp = {"bound": "hbm", "achieved": cmp_bytes / cmp_s / 1e9, "peak": peak, "unit": "GB/s",
                    "frac": cmp_bytes / cmp_s / 1e9 / peak, "traffic": ctraffic,
                    "kernel": "frame_compact_tma_kernel (every valid row once; TMA 2-slot ring per warp, 4-row chunks)",
                    "kernel_ms": 1e3 * cmp_s, "algorithmic_bytes_per_launch": cmp_bytes,
                    "peak_source": peak_src, "traffic_source": ctraffic_src,
                    "share_of_step": cmp_s / (t_dec / args.steps),
                    "note": ("with LM / boosting the pass also issues the decode's L2 warm-up of the lookup tables "
                             "(LM level-1 rows and arcs, boost table) between its rows; those prefetched bytes are "
                             "not counted in algorithmic_bytes_per_launch" if (wl.lm or wl.boost) else None)}

    # e2e through the public host-buffer entry (flexctc_decode_host): H2D + decode + D2H per step
    e2e = None
    if not args.no_e2e:
        Dp = torch.from_numpy(D).to(torch.bfloat16 if bf16 else torch.float32).pin_memory()
        Lp = torch.from_numpy(L).pin_memory()
        nscr = (FX.lib.flexctc_host_scratch_bytes_bf16 if bf16 else FX.lib.flexctc_host_scratch_bytes)(
            B, T, Vp1, __import__("ctypes").byref(cfg))
        scratch = torch.empty(int(nscr), dtype=torch.uint8, device=dev)
        host_decode = F.decode_host_bf16 if bf16 else F.decode_host
        hout = None
        for _ in range(max(1, args.warmup)):
            hout = host_decode(Dp, Lp, cfg, lm, bt, scratch=scratch, stream=stream, out=hout)
        if world > 1:
            dist.barrier()
        ts = []
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            stream.synchronize()
            t0 = time.perf_counter()
            hout = host_decode(Dp, Lp, cfg, lm, bt, scratch=scratch, stream=stream, out=hout)
            ts.append(time.perf_counter() - t0)
        te = torch.tensor([sum(ts)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": frames_all * synth.FRAME_SECONDS * args.steps / float(te[0]), "unit": UNIT,
               # the streamed path (K > 1) copies only the valid frames t < L_b
               "h2d_bytes_per_step": int((int(np.clip(L, 0, T).sum()) * Vp1 * (2 if bf16 else 4) if cfg.beam > 1
                                          else Dp.numel() * Dp.element_size()) + L.nbytes),
               "d2h_bytes_per_step": int(B * T * 4 * 2 + B * 4 * 2),
               "path": (("flexctc_decode_host_bf16 (pinned bf16 logits, 2 B per logit over PCIe; normalised on the "
                         "device per frame chunk" if bf16 else
                         "flexctc_decode_host (pinned host buffers") +
                        "; H2D in frame chunks overlapping the decode, D2H and sync inside)")}

    # gather the final results (the only cross-GPU traffic)
    gathered = None
    if world > 1:
        if strong:
            Btot = int(sum(sh["utterances"] for sh in shards))
            g = gather_results({k: v for k, v in out.items()}, shard_idx, Btot, T, device=dev)
        else:
            g = gather_results({k: v for k, v in out.items()}, np.arange(rank * B, rank * B + B), B * world, T,
                               device=dev)
        gathered = int(g["num_tokens"].sum().item())

    if rank == 0:
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_dec / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "input": args.input,
            "config": workload_config(wl, B, T, frames_local, dict({"parallelism": f"dp{world} (utterance shards)"}
                                      if not strong else
                                      {"parallelism": f"dp{world} (one global batch LPT-sharded by length)",
                                       "global_batch": int(sum(sh["utterances"] for sh in shards)),
                                       "stream_batches": args.stream},
                                      **({"order": "merge-before-TopK (merge_first, R27)"} if args.merge_first else {}))),
            "frames_beams_per_s": fbps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kname, "kernel_ms": 1e3 * kern_s,
                         "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                         "traffic_source": traffic_src,
                         "note": note},
            # our kernels per decode: order_kernel (not on the plain greedy path), l2_warm_kernel (with
            # LM or boost), then the beam kernel (warp path: rowoff + compaction + beam kernel), or
            # frame_summary_kernel + greedy_chain/fused kernel
            "gpu_launches": args.steps * ((0 if plain_greedy else 1) + (1 if (wl.lm or wl.boost) else 0)
                                          + ((3 if compacted else 1) if wl.beam > 1 else 2)),
            "clocks": clk,
            "e2e": e2e,
            "kernel": kernel_name,
            "device_flags": flags,
            "device_stats_per_step": dstats,
        }
        if roof_cmp is not None:
            res["roofline_compact"] = roof_cmp
        if gathered is not None:
            res["gathered_tokens"] = gathered
        if shards is not None:
            mean = sum(fr) / len(fr)
            res["shards"] = shards
            res["load_balance"] = {"max_over_mean_frames": max(fr) / mean if mean else None,
                                   "critical_path_T_max": max(sh["T_max"] for sh in shards),
                                   "slowest_rank_ms": max(sh["ms_per_step"] for sh in shards)}
        if world == 1 and not args.no_cpu_baseline:
            # the whole c4 batch (~20 core-seconds of oracle work); 16 utterances at K = 128
            n = args.cpu_sample or (min(B, 64) if wl.beam <= 32 else min(B, 16))
            res["cpu_baseline"] = cpu_baseline(wl, D, L, arpa, ph, n, int(args.merge_first))
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if world is not None and int(world) != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a mismatched run"}),
              flush=True)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_flexctc(args)


if __name__ == "__main__":
    main()
