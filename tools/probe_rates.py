"""fj_probe_gather at the configs' vector sizes: random-gather rate vs vector rows and width."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

import paper_2101_08143_b200 as fj  # noqa: E402

fj.load_library()
torch.cuda.init()
for n in [1_000_000, 4_000_000, 16_000_000, 67_108_864]:
    for w in [1, 2, 4]:
        if n * w * 8 > 4 << 30:
            continue
        r = fj.probe_gather(n, 64_000_000, width=w, reps=5)
        print(json.dumps({"n_vec": n, "width": w, "MB": n * w * 8 / 1e6, "Ggathers_per_s": r / 1e9}), flush=True)
