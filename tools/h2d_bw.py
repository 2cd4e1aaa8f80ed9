"""H2D bandwidth of pinned host memory on this box: one stream vs two streams (halves of the
same buffer), CUDA events, best of 5. Prints one JSON line (context for the e2e numbers)."""
import json

import torch


def main():
    n = 105 * 1024 * 1024
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, parts in (("1 stream", 1), ("2 streams", 2), ("4 streams", 4)):
        streams = [torch.cuda.Stream() for _ in range(parts)]
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for st in streams:
                st.wait_event(e0)
            step = n // parts
            evs = []
            for i, st in enumerate(streams):
                with torch.cuda.stream(st):
                    d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(st)
                    evs.append(ev)
            for ev in evs:
                torch.cuda.current_stream().wait_event(ev)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res[name] = {"ms": round(best, 3), "GB/s": round(n / best / 1e6, 1)}
    print(json.dumps({"h2d_pinned_105MiB": res}))


if __name__ == "__main__":
    main()
