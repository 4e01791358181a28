"""Where does the host-buffer end-to-end time go?  H2D/D2H link rates and fj_approxim_host phases."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_08143_b200 as fj  # noqa: E402
import synth  # noqa: E402

x = torch.empty(352 << 20, dtype=torch.uint8, pin_memory=True)
y = torch.empty(352 << 20, dtype=torch.uint8, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize()
    print("H2D pinned GB/s", x.numel() / (time.perf_counter() - t) / 1e9, flush=True)
    t = time.perf_counter(); x.copy_(y, non_blocking=True); torch.cuda.synchronize()
    print("D2H pinned GB/s", x.numel() / (time.perf_counter() - t) / 1e9, flush=True)
wl = synth.make_config(sys.argv[1] if len(sys.argv) > 1 else "c3")
uh = torch.from_numpy(wl.u).pin_memory().numpy()
vh = torch.from_numpy(wl.v).pin_memory().numpy()
Sh = torch.from_numpy(wl.S).pin_memory().numpy()
print("pinned?", torch.from_numpy(uh).is_pinned(), uh.dtype, flush=True)
for i in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    z, q, rep = fj.approxim_host(wl.n, uh, vh, None, Sh, want_z=True)
    t1 = time.perf_counter()
    print(f"e2e ms {(t1 - t) * 1e3:.2f}  device approxim ms {rep['ms']:.2f}", flush=True)
