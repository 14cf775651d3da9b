"""Pinned host -> device copy throughput for one 82 MB batch: one copy vs k concurrent chunks."""
import torch
n = 20480000  # C5 batch entries (fp32)
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = (n + k - 1) // k
    main = torch.cuda.current_stream()
    def run():
        ev = torch.cuda.Event()
        ev.record(main)
        for i, s in enumerate(streams):
            s.wait_event(ev)
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            main.wait_stream(s)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{k} chunk(s): {ms:.3f} ms per 81.9 MB -> {4 * n / ms / 1e6:.1f} GB/s")
