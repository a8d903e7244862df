"""Generate the 3-D Legendre golden fixtures tests/golden/p2s3d_*.npz with the
CPU oracle (which tests/test_oracle_reference_pin.py pins to the reference).

  p2s3d_c1.npz      BASELINE config 1 in full: alpha, moments, 64x64 matrix
  p2s3d_vec3.npz    3-component order-3 element pair (Jacobian alpha), full
  p2s3d_c2.npz      configs 2/3/4, one element each: alpha (compact seed),
  p2s3d_c3.npz      row sums, |row| sums and the diagonal of M (the full
  p2s3d_c4.npz      matrices are 2-4 MB each; alpha is regenerated from the
                    seed by the oracle and checked against the stored
                    alpha checksum)

Usage: python tests/golden/make_3d_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1703_09619_b200.configs import CONFIGS  # noqa: E402

SEED = 1703


def main():
    cfg = CONFIGS["c1"]
    o = O.Oracle(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
    a = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, SEED, 0, 1)
    np.savez_compressed(os.path.join(HERE, "p2s3d_c1.npz"), alpha=a, I=o.moments(a), M=o.fill(a),
                        seed=SEED)

    o = O.Oracle(3, (3, 3, 3), [O.PP, O.DD], (6, 6, 6))
    a = o.alpha(O.ALPHA_JACOBIAN, 0.5, 3.0, SEED, 0, 2)
    np.savez_compressed(os.path.join(HERE, "p2s3d_vec3.npz"), alpha=a, I=o.moments(a), M=o.fill(a),
                        seed=SEED)

    for name in ("c2", "c3", "c4"):
        cfg = CONFIGS[name]
        o = O.Oracle(cfg.n_comp, cfg.order, list(cfg.kinds), cfg.nq)
        a = o.alpha(cfg.alpha_kind, cfg.alpha_lo, cfg.alpha_hi, SEED, 7, 1)
        M = o.fill(a, threads=8)[0]
        np.savez_compressed(os.path.join(HERE, f"p2s3d_{name}.npz"), e0=7, seed=SEED,
                            alpha_sum=a.sum(), alpha_abs_sum=np.abs(a).sum(),
                            row_sum=M.sum(axis=1), row_abs_sum=np.abs(M).sum(axis=1),
                            diag=np.diag(M).copy(), first_row=M[0].copy())
    for f in sorted(os.listdir(HERE)):
        if f.startswith("p2s3d_"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
