"""One step of the hot path (fit + run_field) on a workload, for ncu / sanitizer runs.

    python tools/profile_step.py c5 [--reps R]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_12442_b200 import Context, config_args  # noqa: E402
from workloads import generate  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 1
    w = generate(name)
    cfg = w.cfg
    kernel, grid, k, b, hf = config_args(cfg)
    dev = torch.device("cuda:0")
    X = torch.from_numpy(np.array(w.X)).to(dev)
    y = torch.from_numpy(np.array(w.y)).to(dev)
    ctx = Context(0)
    for _ in range(reps):
        ctx.fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf)
        for it, th in enumerate(w.thetas):
            field, n = ctx.run_field(th, cfg.alpha, cfg.max_depth, cfg.n_samples, cfg.mc_seed, it)
    torch.cuda.synchronize()
    print(name, "leaves", n, "field sum", float(field.double().sum()), ctx.stats())


if __name__ == "__main__":
    main()
