"""What plain streaming kernels (torch element-wise ops) reach on this GPU at
the PCG vector sizes: 1R1W copy, 2R1W add, 3R1W addcmul (dev aid; the
practical HBM ceiling for multi-stream kernels like k_pcg_hvp/update)."""
import torch

for n in (1056768, 6316032, 6316032 * 4):
    v = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(5)]
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    ops = {"copy 1R1W": (lambda: v[1].copy_(v[0]), 16),
           "add 2R1W": (lambda: torch.add(v[0], v[1], out=v[2]), 24),
           "addcmul 3R1W": (lambda: torch.addcmul(v[0], v[1], v[2], out=v[3]), 32)}
    for name, (fn, bpe) in ops.items():
        for cold in (False, True):
            ts = []
            for _ in range(20):
                if cold:
                    flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            t = ts[len(ts) // 2] * 1e-3
            print(f"n={n:9d} {name:13s} {'cold' if cold else 'warm'}: {t * 1e6:8.1f} us  {bpe * n / t / 1e9:7.0f} GB/s")
