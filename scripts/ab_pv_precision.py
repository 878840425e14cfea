"""A/B of the P.V operand precision: max / mean error (fp32-output mode) against the fp64 oracle
over seeded mixed batches, for the production library and a variant built with -D flags.
    python scripts/ab_pv_precision.py            (on a GPU box; builds the variants in-tree)"""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = {"rs2_prmt_fadd2": (), "rs1_fhadd": ("PI_P_ROUNDED_SUM=1",), "rs0_exact": ("PI_P_ROUNDED_SUM=0",)}


def child():
    import numpy as np, torch
    from synth import workloads as W
    from tests import gpu_helpers as H
    res = []
    for seed in range(12):
        rng = np.random.default_rng(seed)
        hkv = int(rng.choice([1, 2, 4])); r = int(rng.choice([1, 4, 8]))
        b = W.random_batch(100 + seed, n=int(rng.integers(3, 14)), max_len=int(rng.integers(40, 900)), hq=hkv * r,
                           hkv=hkv, d=128, n_prefix=2)
        t = W.make_tensors(b, device="cuda", peaky=4.0 if seed % 2 else 1.0)   # odd seeds: peaky q (x4)
        out, lse, _ = H.run_batch(b, t, C=int(rng.choice([8192, 512, 200])), delta=2, decode_chunk=256, out_f32=True)
        ro, rl = H.oracle_full(b, t)
        err = np.abs(out.cpu().numpy().astype(np.float64) - ro)
        res.append((float(err.max()), float(err.mean())))
    print(json.dumps({"max": max(x[0] for x in res), "mean": float(np.mean([x[1] for x in res])), "per_seed": res}))


if __name__ == "__main__":
    if "--child" in sys.argv:
        child()
        sys.exit(0)
    from paper_2602_06072_b200 import build as B
    for name, defs in VARIANTS.items():
        lib = B.build(force=True, out=os.path.join(ROOT, "paper_2602_06072_b200", f"libpackinfer_{name}.so"),
                      defines=defs) if defs else B.build()
        env = dict(os.environ, PACKINFER_LIB=lib)
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(name, r.stdout.strip() or r.stderr[-2000:], flush=True)
