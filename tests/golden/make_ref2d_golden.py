"""Generate the reference-pinned golden fixtures tests/golden/ref2d_*.npz.

Runs in the build container only: builds the REFERENCE library from
/root/reference/proj/src with oracle/refbuild/Makefile (outputs into
oracle/_ref/), runs oracle/_ref/ref_probe and stores its output:

  ref2d_quadrature.npz  gauss_legendre(n), n = 1..48      (quadrature.cpp:27-53)
  ref2d_families.npz    eval_T/U/Tns at 32 points, deg<=40 (chebyshev.cpp:23-108)
                        and product_to_sum expansions a,b<=20 (chebyshev.cpp:156-178)
  ref2d_elements.npz    coupling grids + compute_kernel_tables + assemble_p2s_element
                        + assemble_direct_element on the identity element (the KAT of
                        test_assembly.cpp:96-140) and seeded curved elements (seeds 57/91,
                        test_assembly.cpp:142-172)

Usage: python tests/golden/make_ref2d_golden.py
"""
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle", "refbuild"), "-s"], check=True)
    out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_probe")], check=True,
                         capture_output=True, text=True).stdout
    d = json.loads(out)

    q = {}
    for r in d["quadrature"]:
        q[f"nodes_{r['n']}"] = np.array(r["nodes"])
        q[f"weights_{r['n']}"] = np.array(r["weights"])
    np.savez_compressed(os.path.join(HERE, "ref2d_quadrature.npz"), **q)

    # p2s rows: fa, a, fb, b, then (coeff, family, degree) * n_terms; pad to 2 terms
    rows = np.zeros((len(d["p2s"]), 4 + 6))
    nterm = np.zeros(len(d["p2s"]), dtype=np.int64)
    for i, r in enumerate(d["p2s"]):
        rows[i, :len(r)] = r
        nterm[i] = (len(r) - 4) // 3
    np.savez_compressed(os.path.join(HERE, "ref2d_families.npz"), points=np.array(d["points"]),
                        values=np.array(d["family_values"]).reshape(3, 41, -1), p2s=rows,
                        p2s_nterms=nterm)

    el = {}
    tags = []
    for c in d["cases"]:
        tag = c["tag"]
        tags.append(tag)
        for k in ("M", "N", "nq", "geom_order", "n_integrals", "n_mass_uu_integrals",
                  "direct_n_integrals"):
            el[f"{tag}__{k}"] = np.array(c[k])
        el[f"{tag}__nodes"] = np.array(c["nodes"])
        for k, v in c.items():
            if isinstance(v, dict) and "rows" in v:
                el[f"{tag}__{k}"] = np.array(v["data"]).reshape(v["rows"], v["cols"])
    el["tags"] = np.array(tags)
    # conforming_matrix(d), d = 1..16 (n = d + 1), row-major
    for d_, r in enumerate(d["conforming"], start=1):
        el[f"conforming_matrix__{d_ + 1}"] = np.array(r).reshape(d_ + 1, d_ + 1)
    np.savez_compressed(os.path.join(HERE, "ref2d_elements.npz"), **el)
    for f in ("ref2d_quadrature.npz", "ref2d_families.npz", "ref2d_elements.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
