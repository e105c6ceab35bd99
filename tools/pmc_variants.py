"""k_pmc tuning harness: build liblcp.so variants with different compile-time
knobs of pmc.cu, then time the MC kernel of each on the same c5 leaf chunk.

    python tools/pmc_variants.py build NAME "-DPMC_MINBLOCKS=3 -DPMC_ILP=2" [...]
    python tools/pmc_variants.py run   [--cells 4194304] NAME [NAME ...]   (GPU)

Variants live under variants/NAME/liblcp.so (git-ignored).  `run` loads each in
a fresh subprocess (LCP_LIB) and prints one line per variant: MC ms, samples/s,
phase-2 fraction, and an LCP checksum that must agree across variants that
claim identical arithmetic.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(name, flags):
    from paper_2512_12442_b200 import _build as B
    B.build()
    out = os.path.join(ROOT, "variants", name)
    os.makedirs(out, exist_ok=True)
    obj = os.path.join(out, "pmc.cu.o")
    cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *flags.split(), "-Xptxas", "-v", "-c",
           os.path.join(B.CSRC, "pmc.cu"), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    regs, cur = [], None
    for line in r.stderr.splitlines():
        if "Compiling entry function" in line:
            cur = line.split("'")[1]
        elif "Used" in line and cur and "k_pmcILi1E" in cur:
            regs.append(line.strip())
        elif "spill" in line and cur and "k_pmcILi1E" in cur:
            regs.append(line.strip())
    objs = [os.path.join(B.BUILD, f) for f in sorted(os.listdir(B.BUILD))
            if f.endswith(".o") and f != "pmc.cu.o"] + [obj]
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", os.path.join(out, "liblcp.so"), *objs, "-lcudart"])
    print(name, flags, "|", " ; ".join(regs[:12]))


def run_one(n_cells):
    import numpy as np
    import torch
    from paper_2512_12442_b200 import Context, config_args
    from workloads import generate
    w = generate("c5")
    cfg = w.cfg
    kernel, grid, k, b, hf = config_args(cfg)
    dev = torch.device("cuda:0")
    X = torch.from_numpy(np.array(w.X)).to(dev)
    y = torch.from_numpy(np.array(w.y)).to(dev)
    ctx = Context(0).fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf)
    th = w.thetas[0]
    leaves = ctx.octree_refine(th, cfg.alpha, cfg.max_depth)[:n_cells].clone()
    out = torch.empty(len(leaves), dtype=torch.float32, device=dev)
    best = None
    for _ in range(4):
        ctx.pmc_cells(leaves, th, cfg.n_samples, cfg.mc_seed, 0, out=out)
        torch.cuda.synchronize()
        st = ctx.stats()
        best = st if best is None or st["mc_ms"] < best["mc_ms"] else best
    samples = len(leaves) * cfg.n_samples
    print(json.dumps({"lib": os.environ.get("LCP_LIB", "default"), "mc_ms": best["mc_ms"],
                      "samples_per_s": samples / (best["mc_ms"] / 1e3),
                      "phase2_frac": best["pmc_phase2_samples"] / samples,
                      "checksum": float(out.double().sum())}), flush=True)


def main():
    mode = sys.argv[1]
    if mode == "build":
        build(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
    elif mode == "one":
        run_one(int(sys.argv[2]))
    else:
        args = sys.argv[2:]
        n = 1 << 22
        if args and args[0] == "--cells":
            n = int(args[1])
            args = args[2:]
        for name in args:
            env = dict(os.environ)
            if name != "default":
                env["LCP_LIB"] = os.path.join(ROOT, "variants", name, "liblcp.so")
            subprocess.run([sys.executable, __file__, "one", str(n)], env=env)


if __name__ == "__main__":
    main()
