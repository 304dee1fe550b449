"""H2D bandwidth: one 40 MB copy vs the same bytes split over K streams."""
import torch
mb = 40
n = mb * 2**20 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for k in (1, 2, 4, 8):
    chunk = (n + k - 1) // k
    def run():
        cur = torch.cuda.current_stream()
        for i in range(k):
            s = streams[i]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for i in range(k):
            cur.wait_stream(streams[i])
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"k={k}: {ms:.3f} ms = {mb * 2**20 / ms / 1e6:.1f} GB/s")
