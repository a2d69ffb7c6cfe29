"""Regenerate the batch-scale golden fixtures from the REFERENCE build (oracle/_ref):

  tests/golden/config2_full.json    all 1,024 config-2 points (config-1 network, F from
                                    the mt19937_64(55) recipe, stress only): status, base
                                    iterations, sigma, and the polar stretch U
  tests/golden/config5_sample.json  64 config-5 points (config-3 networks p = 64 k, base +
                                    6 warm probes + tangent): status, iterations, solves,
                                    sigma, spatial C
  tests/golden/config3_sample.json  (with --config3-ids FILE) the listed config-3 points,
                                    stress only

Every DR solve and homogenized stress is the reference's own compiled relax_solve /
homogenized_stress (ref_shim.cpp ref_batch_response, WorkerPool over all host cores); the
networks come from the reference's own generator; the Eigen-dependent tensor steps use the
oracle's Eigen 3.4.0 restatement.  Run here, where /root/reference exists (minutes of CPU):

  python tests/golden/make_golden_batches.py [--config3-ids ids.txt]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402
from oracle import workload as W  # noqa: E402


def hexs(a):
    return [float(x).hex() for x in np.asarray(a).ravel()]


def records(out, idx, extra=None):
    rows = []
    for i, p in enumerate(idx):
        r = {"p": int(p), "status": int(out["status"][i]),
             "base_iterations": int(out["base_iterations"][i]),
             "relax_iterations": int(out["relax_iterations"][i]),
             "solves": int(out["solves"][i]), "failed_probe": int(out["failed_probe"][i]),
             "sigma": hexs(out["sigma"][i])}
        if extra:
            r.update(extra(i))
        rows.append(r)
    return rows


def config2(workers):
    rnet = O.ref_generate(seed=W.NET_SEED, **W.CONFIG1_KNN)
    F = W.batch_F(1024).reshape(1024, 9)
    t0 = time.time()
    out = O.ref_batch_response([rnet], np.zeros(1024, np.int32), F, want_tangent=False,
                               workers=workers)
    U = [O.polar_decompose(F[p])[1] for p in range(1024)]
    print(f"config2: {time.time() - t0:.0f} s, failed {int((out['status'] != 0).sum())}")
    return {"network": dict(W.CONFIG1_KNN, seed=W.NET_SEED), "F": "oracle/workload.py batch_F(1024)",
            "points": records(out, range(1024), lambda i: {"U": hexs(U[i])})}


def config_sample(points, tangent, workers):
    nets, seeds = zip(*[W.config3_ref_network(int(p)) for p in points])
    F = W.batch_F(max(points) + 1).reshape(-1, 9)[list(points)]
    t0 = time.time()
    out = O.ref_batch_response(list(nets), np.arange(len(points), dtype=np.int32), F,
                               want_tangent=tangent, workers=workers)
    print(f"{len(points)} config-3 networks tangent={tangent}: {time.time() - t0:.0f} s, "
          f"failed {int((out['status'] != 0).sum())}")
    extra = (lambda i: {"seed": int(seeds[i]), "spatial_c": hexs(out["spatial_c"][i])}) if tangent \
        else (lambda i: {"seed": int(seeds[i])})
    return {"networks": "oracle/workload.py config3_spec(p), reference generator",
            "F": "rows p of batch_F(16384)", "tangent": tangent,
            "points": records(out, points, extra)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", choices=["config2", "config5", "config3"], default=None)
    ap.add_argument("--config3-ids", default=None)
    a = ap.parse_args()
    O.build(ref=True)
    workers = os.cpu_count() or 1
    jobs = []
    if a.only in (None, "config2"):
        jobs.append(("config2_full.json", lambda: config2(workers)))
    if a.only in (None, "config5"):
        jobs.append(("config5_sample.json",
                     lambda: config_sample(list(range(0, 4096, 64)), True, workers)))
    if a.config3_ids and a.only in (None, "config3"):
        ids = sorted({int(x) for x in open(a.config3_ids).read().split()})
        jobs.append(("config3_sample.json", lambda: config_sample(ids, False, workers)))
    for name, fn in jobs:
        data = fn()
        with open(os.path.join(HERE, name), "w") as fh:
            json.dump(data, fh, separators=(",", ":"))
        print("wrote", name)


if __name__ == "__main__":
    main()
