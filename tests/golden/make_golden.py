"""Generate the committed golden fixtures from the COMPILED REFERENCE
(oracle/_ref/libparcop_ref.so = /root/reference/proj/include/parcop built in
place with oracle/shim.hpp). Run in the build container:

    python tests/golden/make_golden.py

Fixtures:
  c1_gaussian_rho05_n1e4.npz  configs[0] input: the reference's own
                              sample_matrix (RngStream / mt19937_64) at
                              Gaussian rho=0.5, n=1e4, seed mix_seed(B,{0,1e4,10,0})
  c1_expected.json            per-block FitResult + combined theta from the
                              reference headers + SPEC driver; sha256 of the
                              reference's segment-local ranks
  points.json                 log_pdf / shc of the reference at 270 points
  ranks_small.json            rank vectors of the reference on small columns
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import BASE_SEED, ref_lib  # noqa: E402


def main():
    ref = ref_lib()
    assert ref is not None, "build oracle/_ref first (make -C oracle)"
    n, k = 10000, 10
    seed = ref.lib.ref_mix_seed4(BASE_SEED, 0, n, k, 0)
    c1, c2 = ref.sample_matrix(0, 0.5, n, seed)
    np.savez_compressed(os.path.join(HERE, "c1_gaussian_rho05_n1e4.npz"), col1=c1, col2=c2)
    off = ref.partition(n, k)
    recs = ref.fit_blocks(0, c1, c2, off, workers=4)
    tc, w, used = ref.combine(recs)
    u1 = np.concatenate([ref.rank_column(c1[int(off[m]):int(off[m + 1])]) for m in range(k)])
    u2 = np.concatenate([ref.rank_column(c2[int(off[m]):int(off[m + 1])]) for m in range(k)])
    meta = {
        "config": "Gaussian rho=0.5, n=1e4, K=10 (BASELINE.json configs[0])",
        "seed": int(seed),
        "per_block": [{"theta_hat": r.theta_hat, "sigma2": r.sigma2, "loglik": r.loglik, "n": int(r.n),
                       "converged": int(r.converged)} for r in recs],
        "theta_combined": tc,
        "weights": w.tolist(),
        "blocks_used": int(used),
        "ranks_sha256": hashlib.sha256(u1.tobytes() + u2.tobytes()).hexdigest(),
    }
    json.dump(meta, open(os.path.join(HERE, "c1_expected.json"), "w"), indent=1)

    rng = np.random.default_rng(1609)
    pts = []
    models = [(0, 0.0), (0, 0.3), (0, -0.8), (0, 0.95), (1, 5.0), (1, -3.0), (1, 0.5), (1, 20.0), (2, 1.0),
              (2, 2.0), (2, 5.0), (2, 12.0)]
    uv = np.r_[rng.uniform(0.001, 0.999, (20, 2)), [[1e-6, 0.5], [0.5, 1 - 1e-6], [0.3, 0.3], [0.999, 0.998],
                                                 [1e-5, 1e-5], [0.5, 0.5]]]
    for fam, th in models:
        lp = ref.log_pdf(fam, th, uv[:, 0], uv[:, 1])
        d = ref.derivs(fam, th, uv[:, 0], uv[:, 1])
        for i in range(len(uv)):
            pts.append({"family": fam, "theta": th, "u": uv[i, 0], "v": uv[i, 1], "log_pdf": lp[i],
                        "score": d[i, 0], "hess": d[i, 1], "cross1": d[i, 2], "cross2": d[i, 3]})
    json.dump(pts, open(os.path.join(HERE, "points.json"), "w"))

    cols = {
        "spec_example": [3.1, 1.2, 7.5],
        "spec_ties": [1.0, 1.0, 2.0],
        "signed_zero": [0.0, -0.0, 1.0, -1.0, -0.0],
        "runs": [2.0, 1.0, 2.0, 2.0, 1.0, 3.0, 0.5, 3.0],
        "random50": np.round(rng.standard_normal(50), 1).tolist(),
    }
    out = {name: {"x": c, "u": ref.rank_column(np.array(c, np.float64)).tolist()} for name, c in cols.items()}
    json.dump(out, open(os.path.join(HERE, "ranks_small.json"), "w"), indent=1)
    print("golden fixtures written; theta_combined", tc)


if __name__ == "__main__":
    main()
