"""Effective bandwidth of torch copy (read + write) vs working-set size on one B200: where L2
residency stops paying.  Prints one JSON line per size."""
import json
import torch

torch.cuda.set_device(0)
for mb in [8, 16, 32, 48, 64, 96, 128, 256, 1024, 4096]:
    n = mb * 2**20 // 8 // 2
    a = torch.randn(n, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    for _ in range(5):
        b.copy_(a)
    reps = max(20, int(2000 / mb))
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    # read-only: sum
    for _ in range(3):
        a.sum()
    e0.record()
    for _ in range(reps):
        a.sum()
    e1.record()
    torch.cuda.synchronize()
    tr = e0.elapsed_time(e1) / reps / 1e3
    print(json.dumps({"working_set_MB": mb, "copy_GBps": round(2 * n * 8 / t / 1e9, 1), "copy_us": round(t * 1e6, 2),
                      "sum_read_GBps": round(n * 8 / tr / 1e9, 1)}), flush=True)
