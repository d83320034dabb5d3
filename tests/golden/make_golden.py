"""Generate tests/golden/* from the UNMODIFIED reference (oracle/_ref/librsvd_ref.so).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The outputs are committed; the GPU box never needs the reference itself.

Contents
  golden.json   Philox words/units/gaussians, gen_sketch arrays for every
                reference kind, and run_fixed_precision / run_fixed_rank
                results (rank, blocks, ids, per-block residuals, sigma).
  matrices.npz  the small test matrices those runs used (reference
                gen_synthetic, SlowDecay/FastDecay, stored as float64).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Oracle  # noqa: E402

KINDS = {"gaussian": 0, "bernoulli": 1, "stdbernoulli": 2, "sparsesign": 3, "sparsegaussian": 4}


def main():
    R = Oracle("reference")
    g = {"philox": [], "sketch": [], "runs": []}
    for seed, blk, col in [(0, 0, 0), (42, 0, 0), (42, 3, 17), (7, 1000, 5), (2**40 + 3, 2, 1)]:
        g["philox"].append({
            "seed": seed, "block_id": blk, "column": col,
            "u32": [int(x) for x in R.philox_u32(seed, blk, col, 16)],
            "units": [float(x) for x in R.philox_units(seed, blk, col, 8)],
            "gaussians": [float(x) for x in R.philox_gaussians(seed, blk, col, 9)],
        })
    cases = [
        ("sparsesign", 4e-4, 42, 20000, 4, 0),
        ("bernoulli", 4e-4, 42, 20000, 4, 0),
        ("sparsegaussian", 4e-4, 42, 20000, 4, 0),
        ("stdbernoulli", 0.05, 9, 500, 7, 3),
        ("sparsesign", 0.1, 7, 500, 40, 0),
        ("sparsegaussian", 0.1, 7, 500, 40, 1000),
        ("stdbernoulli", 0.5, 11, 300, 5, 2),
        ("gaussian", 0.0, 5, 64, 3, 1),
    ]
    for name, p, seed, n, l, bid in cases:
        s = R.gen_sketch(KINDS[name], p, seed, n, l, bid)
        e = {"kind": name, "p": p, "seed": seed, "n": n, "l": l, "block_id": bid}
        if s.is_dense:
            e["dense"] = s.dense.flatten(order="F").tolist()
        else:
            e.update(col_ptr=s.col_ptr.tolist(), row_idx=s.row_idx.tolist(),
                     values=s.values.tolist(), centered=s.centered, std_scale=s.std_scale)
        g["sketch"].append(e)

    mats = {
        "slow128": R.gen_synthetic(0, 128, 5),
        "fast96": R.gen_synthetic(1, 96, 68),
        "slow200": R.gen_synthetic(0, 200, 64),
    }
    np.savez_compressed(os.path.join(HERE, "matrices.npz"), **mats)
    runs = []
    for mat in ("slow128", "fast96"):
        for kind in KINDS:
            for power in (0, 1, 2, 3):
                p = 0.0 if kind == "gaussian" else 0.08
                # slow128 reaches 1e-2 (rank ~16); fast96 cannot reach 1e-3 within
                # max_iters and exercises the ToleranceNotReached partial result.
                runs.append(dict(matrix=mat, kind=kind, p=p, power=power, block=8, seed=61,
                                 eps=1e-2 if mat == "slow128" else 1e-3, relative=True, rank=None))
    runs.append(dict(matrix="slow200", kind="stdbernoulli", p=0.05, power=1, block=20, seed=65,
                     eps=0, relative=True, rank=60))
    runs.append(dict(matrix="slow128", kind="gaussian", p=0.0, power=1, block=10, seed=79,
                     eps=0, relative=True, rank=25))
    runs.append(dict(matrix="slow128", kind="gaussian", p=0.0, power=1, block=10, seed=77,
                     eps=1e-6, relative=True, rank=None, max_iters=2))
    for r in runs:
        a = mats[r["matrix"]]
        res = R.run(a, eps=r["eps"], power=r["power"], block=r["block"], kind=KINDS[r["kind"]],
                    p=r["p"], seed=r["seed"], relative=r["relative"], rank=r["rank"],
                    max_iters=r.get("max_iters", 0), traced=True)
        r.update(status=res.status, out_rank=res.rank, blocks=res.blocks,
                 converged=res.converged, residual_sq=res.residual_sq,
                 norm_a_sq=res.norm_a_sq, sigma=res.sigma.tolist(),
                 block_ids=res.block_ids, block_residuals=res.block_residuals.tolist())
        g["runs"].append(r)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=0)
    print("wrote", len(g["runs"]), "runs")


if __name__ == "__main__":
    main()
