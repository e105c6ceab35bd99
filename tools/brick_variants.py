"""k_brick tuning harness: build liblcp.so variants with compile-time knobs of brick.cu,
then time the c5 refine-time brick pass of each (fit + refine, best of 3).

    python tools/brick_variants.py build NAME "-DBRICK_UNROLL=8" [...]
    python tools/brick_variants.py run NAME [NAME ...]          (GPU; "default" = the in-tree build)
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
    obj = os.path.join(out, "brick.cu.o")
    cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *flags.split(), "-Xptxas", "-v", "-c", os.path.join(B.CSRC, "brick.cu"),
           "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    info = [ln.strip() for ln in r.stderr.splitlines() if "Used" in ln or "spill" in ln]
    objs = [os.path.join(B.BUILD, f) for f in sorted(os.listdir(B.BUILD))
            if f.endswith(".o") and f != "brick.cu.o"] + [obj]
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", os.path.join(out, "liblcp.so"), *objs, "-lcudart"])
    print(name, flags, "|", " ; ".join(info[:6]))


def run_one():
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
    ctx = Context(0)
    best = None
    from paper_2512_12442_b200 import LcpError
    diag = False
    for _ in range(3):
        ctx.fit_local(X, y, kernel, k, grid, bucket_log2=b, h_full=hf)
        try:
            leaves = ctx.octree_refine(w.thetas[0], cfg.alpha, cfg.max_depth)
        except LcpError:   # BRICK_DIAG_* timing variants write invalid posteriors
            diag = True
        st = ctx.stats()
        best = st if best is None or st["brick_pass_ms"] < best["brick_pass_ms"] else best
    if diag:
        print(json.dumps({"lib": os.environ.get("LCP_LIB", "default"), "brick_pass_ms": best["brick_pass_ms"],
                          "refine_ms": best["refine_ms"], "diag": True}), flush=True)
        return
    sub = leaves[: 1 << 20].clone()
    lcp = ctx.pmc_cells(sub, w.thetas[0], 1024, cfg.mc_seed)
    print(json.dumps({"lib": os.environ.get("LCP_LIB", "default"), "brick_pass_ms": best["brick_pass_ms"],
                      "refine_ms": best["refine_ms"], "leaves": int(len(leaves)),
                      "checksum": float(lcp.double().sum())}), flush=True)


def main():
    mode = sys.argv[1]
    if mode == "build":
        build(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
    elif mode == "one":
        run_one()
    else:
        for name in sys.argv[2:]:
            env = dict(os.environ)
            if name != "default":
                env["LCP_LIB"] = os.path.join(ROOT, "variants", name, "liblcp.so")
            subprocess.run([sys.executable, __file__, "one"], env=env)


if __name__ == "__main__":
    main()
