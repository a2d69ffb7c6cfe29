"""Regenerate tests/golden/*.json from the REFERENCE build (oracle/_ref, the reference's own
network.cpp / relax.cpp / netgen.cpp compiled from /root/reference).  Run here, where the
reference sources exist:  python tests/golden/make_golden.py

The fixtures pin the oracle restatement (and, through it, the GPU parity tests) to the
reference's own outputs on the GPU box, where /root/reference is absent.  Floating-point
values are stored as hex bit patterns so bitwise comparisons survive JSON.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402
from paper_2306_09427_b200.synth import batch_F  # noqa: E402


def h64(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hexf(x):
    return float(x).hex()


NETS = [  # (style, kwargs, seed) -- the reference tests' specs + the config-1 network
    ("knn", dict(nodes=16, fibers=44, neighbors=10), 11),
    ("knn", dict(nodes=16, fibers=44, neighbors=10), 21),
    ("knn", dict(nodes=20, fibers=56, neighbors=10), 31),
    ("knn", dict(nodes=14, fibers=38, neighbors=9), 101),
    ("knn", dict(nodes=12, fibers=32, neighbors=9), 102),
    ("knn", dict(nodes=375, fibers=1000, neighbors=10), 1),
    ("knn", dict(nodes=375, fibers=1000, neighbors=10), 4),
    ("segments", dict(fibers=200), 5),
    ("knn", dict(nodes=60, fibers=200, neighbors=8, align_bias=2.0, align_axis=(1.0, 1.0, 0.0)), 4),
]

SOLVES = [  # (net index, F) -- diagonal loads so the polar step is exact everywhere
    (2, [1.06, 1.0, 0.97]),
    (0, [1.04, 0.99, 1.01]),
    (3, [1.02, 1.0, 1.0]),
    (6, [1.05, 1.0, 1.0]),
    (5, [1.25, 1.0, 1.0]),
]


def main():
    O.build(ref=True)
    out = {"generator": [], "relax": [], "batch_F": {}}
    for style, kw, seed in NETS:
        rn = O.ref_generate(style, seed=seed, **kw)
        out["generator"].append({
            "style": style, "spec": kw, "seed": seed, "n_nodes": rn.n_nodes,
            "n_fibers": rn.n_fibers, "n_free": rn.n_free, "n_boundary": rn.n_boundary,
            "coords_sha256": h64(rn.coords), "fibers_sha256": h64(np.stack([rn.fib_a, rn.fib_b])),
            "packed_of_dof_sha256": h64(rn.packed_of_dof), "fiber_dofs_sha256": h64(rn.fiber_dofs),
            "node_lump_sha256": h64(rn.node_lump), "rest_length_sha256": h64(rn.rest_length),
        })
    for ni, diag in SOLVES:
        style, kw, seed = NETS[ni]
        rn = O.ref_generate(style, seed=seed, **kw)
        F = np.diag(diag)
        st, rep = O.ref_relax_solve(rn, F)
        sig, asym = O.ref_homogenized_stress(rn, st, F) if rep["converged"] else (np.zeros(6), 0.0)
        out["relax"].append({
            "net": ni, "F_diag": diag, "iterations": rep["iterations"],
            "converged": rep["converged"],
            "residual": hexf(rep["residual"]), "eps_eff": hexf(rep["eps_eff"]),
            "kinetic_fraction": hexf(rep["kinetic_fraction"]), "dt": hexf(rep["dt"]),
            "t": hexf(st.t[0]),
            "u_sha256": h64(st.u), "v_sha256": h64(st.v), "f_int_sha256": h64(st.f_int),
            "sigma": [hexf(x) for x in sig], "asym": hexf(asym),
        })
    F = batch_F(16)
    out["batch_F"] = {"n": 16, "seed": 55, "sha256": h64(F)}
    with open(os.path.join(HERE, "reference_fixtures.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", os.path.join(HERE, "reference_fixtures.json"))


if __name__ == "__main__":
    main()
