"""Experiment helper (GPU box): PCIe copy throughput from pinned host memory,
one copy per direction against copies split over several streams, alone and
with the other direction running (duplex)."""
import torch

nb = 1 << 30
h_in = torch.empty(nb // 8, dtype=torch.float64).pin_memory()
h_out = torch.empty(nb // 8, dtype=torch.float64).pin_memory()
d_in = torch.empty(nb // 8, dtype=torch.float64, device="cuda")
d_out = torch.empty(nb // 8, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(h2d_split, d2h_split, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        used = []
        for i in range(h2d_split):
            s = streams[i]
            s.wait_event(e0)
            c = nb // 8 // h2d_split
            with torch.cuda.stream(s):
                d_in[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
            used.append(s)
        for i in range(d2h_split):
            s = streams[4 + i]
            s.wait_event(e0)
            c = nb // 8 // d2h_split
            with torch.cuda.stream(s):
                h_out[i * c:(i + 1) * c].copy_(d_out[i * c:(i + 1) * c], non_blocking=True)
            used.append(s)
        for s in used:
            ev = torch.cuda.Event()
            ev.record(s)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for hs, ds in ((1, 0), (2, 0), (4, 0), (0, 1), (0, 2), (0, 4), (1, 1), (2, 2), (4, 4)):
    ms = run(hs, ds)
    print(f"H2D x{hs} D2H x{ds}: {ms:.2f} ms  -> {nb / ms / 1e6:.1f} GB/s per active direction")
