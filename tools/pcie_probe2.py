"""D2H copy bandwidth of per-frame output downloads: three copies (quad 4.9 MB, depth 1.2 MB,
weight 1.2 MB) against one 7.4 MB copy per frame, 300 frames, 1 and 8 streams (timing
experiment, not the bench)."""
import torch

W, H = 640, 480
plane = W * H
d = torch.empty(32 * 8 * plane, dtype=torch.float32, device="cuda")
h = torch.empty(300 * 6 * plane, dtype=torch.float32).pin_memory()
for nstreams in (1, 8):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    for mode in ("3 copies", "1 copy"):
        def run():
            for f in range(300):
                s = streams[f % nstreams]
                src = d[(f % 32) * 8 * plane:]
                dst = h[f * 6 * plane:]
                with torch.cuda.stream(s):
                    if mode == "1 copy":
                        dst[:6 * plane].copy_(src[:6 * plane], non_blocking=True)
                    else:
                        dst[:4 * plane].copy_(src[:4 * plane], non_blocking=True)
                        dst[4 * plane:5 * plane].copy_(src[5 * plane:6 * plane], non_blocking=True)
                        dst[5 * plane:6 * plane].copy_(src[6 * plane:7 * plane], non_blocking=True)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        for s in streams:
            e1.wait_stream(s) if hasattr(e1, "wait_stream") else None
        torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        import time
        t0 = time.perf_counter()
        run()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        gb = 300 * 6 * plane * 4 / 1e9
        print(f"{nstreams} streams, {mode}: {gb / dt:.1f} GB/s ({300 / dt:.0f} frames/s)", flush=True)
