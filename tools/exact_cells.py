"""How many leaf cells have an MC count fixed by worst-case bounds (every sample
all-below, all-above, or crossing), so that sampling them is unnecessary?
Bound: |z_d| <= 5.7684 for every normal Box-Muller can produce (u >= 2^-24), so
y_c lies in [mu_c - Z ||L_c||_1, mu_c + Z ||L_c||_1] for every sample.

    python tools/exact_cells.py c5 p1 c3      (GPU)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2512_12442_b200 import Context, config_args
    from workloads import generate
    Z = 5.7684
    for name in sys.argv[1:]:
        w = generate(name)
        cfg = w.cfg
        kernel, grid, k, b, hf = config_args(cfg)
        dev = torch.device("cuda:0")
        ctx = Context(0).fit_local(torch.from_numpy(np.array(w.X)).to(dev), torch.from_numpy(np.array(w.y)).to(dev),
                                   kernel, k, grid, bucket_log2=b, h_full=hf)
        th = w.thetas[0]
        leaves = ctx.octree_refine(th, cfg.alpha, cfg.max_depth)
        sel = torch.from_numpy(np.random.default_rng(0).choice(len(leaves), min(20000, len(leaves)), replace=False)).to(dev)
        mu, cov = ctx.cell_posterior(leaves[sel].contiguous())
        mu, cov = mu.cpu().numpy(), cov.cpu().numpy()
        n_below = n_above = n_cross = 0
        for q in range(len(mu)):
            S = cov[q]
            # clamped Cholesky as the library does (PSD clamp)
            try:
                L = np.linalg.cholesky(S + 1e-14 * np.eye(8) * np.trace(S))
            except np.linalg.LinAlgError:
                continue
            r = Z * np.abs(L).sum(axis=1)
            lo, hi = mu[q] - th - r, mu[q] - th + r
            if np.all(hi < 0):
                n_below += 1
            elif np.all(lo > 0):
                n_above += 1
            elif np.any(hi < 0) and np.any(lo > 0):
                n_cross += 1
        n = len(mu)
        print(f"{name}: {len(leaves)} leaves, sample {n}: all-below {n_below / n:.4f}, all-above {n_above / n:.4f}, "
              f"always-crossing {n_cross / n:.4f}")


if __name__ == "__main__":
    main()
