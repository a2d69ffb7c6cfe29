"""Shared helpers: the same synthetic network as product object and oracle object."""
import numpy as np

import oracle as O
import paper_2306_09427_b200 as P
from paper_2306_09427_b200.synth import batch_F


def pair(seed, **spec):
    pn = P.generate_network(P.NetGenSpec(**spec), seed)
    on = O.Network(pn.coords, pn.fiber_nodes[:, 0], pn.fiber_nodes[:, 1], pn.fiber_area,
                   pn.fiber_modulus, pn.box_half)
    return pn, on


def knn(nodes, fibers, seed, neighbors=10):
    return pair(seed, style="knn", nodes=nodes, fibers=fibers, neighbors=neighbors)


def bits(x):
    x = np.ascontiguousarray(x)
    return x.view(np.uint64) if x.dtype == np.float64 else x


def same_bits(a, b):
    return np.array_equal(bits(np.asarray(a, dtype=np.float64)), bits(np.asarray(b, dtype=np.float64)))


def oracle_batch(onets, eop, F, relax=None, law=None, tangent=True, threads=8):
    st = O.PackedStates.fresh(onets, eop)
    resp, status = O.batch_response(onets, eop, st, F, relax_cfg=relax, law=law,
                                    want_tangent=tangent, n_threads=threads)
    return resp, status, st


__all__ = ["pair", "knn", "bits", "same_bits", "oracle_batch", "batch_F"]
