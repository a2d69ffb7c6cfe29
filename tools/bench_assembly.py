"""Bench of the device macro assembly (csrc/assembly.cu).

Workload: a make_box_mesh(N, N, N) macro mesh (6 N^3 linear tets), xmin pinned (affine)
and zmax z set, coords perturbed, one response record per tet (sigma + Mandel C) -- the
consumer step of batch_response in a macro Newton iteration (macrofem.cpp:104-187).
Prints one JSON line like bench.py: ``value`` = assembled tets/s with inputs in HBM (CUDA
events on the assembler's stream, L2 flushed between steps), ``e2e`` through the host
call (H2D of coords/responses, D2H of residual + values inside the timed region),
``roofline`` against the measured HBM peak with the algorithmic bytes (responses, tets,
coords, the compressed values, the residual) and the per-kernel split, and
``cpu_baseline`` = the oracle's C restatement (one thread) on a bounded mesh.

    python tools/bench_assembly.py [--cells 60] [--steps 5] [--warmup 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make_case(n, seed=1):
    from paper_2306_09427_b200.assembly import DirichletBc, build_numbering, make_box_mesh
    rng = np.random.default_rng(seed)
    mesh = make_box_mesh(n, n, n)
    mesh.coords = mesh.ref_coords + rng.uniform(-0.05 / n, 0.05 / n, mesh.ref_coords.shape)
    num = build_numbering(mesh, [DirichletBc("xmin", affine=np.eye(3)),
                                 DirichletBc("zmax", value=(None, None, 0.0))])
    ne = mesh.n_elements
    resp = np.empty((ne, 42))
    resp[:, :6] = rng.standard_normal((ne, 6))
    resp[:, 6:] = rng.standard_normal((ne, 36))
    return mesh, num, resp


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=60)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-cells", type=int, default=16)
    args = ap.parse_args()
    import torch

    from paper_2306_09427_b200.assembly import MacroAssembler
    dev = torch.device("cuda:0")
    t0 = time.time()
    mesh, num, resp = make_case(args.cells)
    A = MacroAssembler(mesh, num)
    plan_s = time.time() - t0
    info = A.info()
    ne, nnz, nf = mesh.n_elements, A.nnz, num.n_free
    d_x = torch.from_numpy(np.ascontiguousarray(mesh.coords)).to(dev)
    d_r = torch.from_numpy(resp).to(dev)
    d_res = torch.empty(nf, dtype=torch.float64, device=dev)
    d_val = torch.empty(nnz, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)
    A.set_stream(stream.cuda_stream)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        A.assemble_device(d_x.data_ptr(), d_r.data_ptr(), 42, None, d_res.data_ptr(),
                          d_val.data_ptr())
    A.status()
    tot, parts = 0.0, np.zeros(3)
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        A.assemble_device(d_x.data_ptr(), d_r.data_ptr(), 42, None, d_res.data_ptr(),
                          d_val.data_ptr())
        ev1.record(stream)
        A.status()
        tot += ev0.elapsed_time(ev1)
        parts += np.array(A.times_ms())
    ms = tot / args.steps
    parts /= args.steps
    # e2e through the host call (pinned buffers)
    x_h = torch.from_numpy(np.ascontiguousarray(mesh.coords)).pin_memory().numpy()
    r_h = torch.from_numpy(resp).pin_memory().numpy()
    o_h = (torch.empty(nf, dtype=torch.float64).pin_memory().numpy(),
           torch.empty(nnz, dtype=torch.float64).pin_memory().numpy())
    A.assemble(x_h, responses=r_h, stride=42, out=o_h)
    t = time.perf_counter()
    for _ in range(args.steps):
        A.assemble(x_h, responses=r_h, stride=42, out=o_h)
    e2e_ms = (time.perf_counter() - t) * 1e3 / args.steps
    # algorithmic bytes: responses + tets + coords in, compressed values + residual out
    alg = ne * (42 * 8 + 16) + mesh.n_nodes * 24 + nnz * 8 + nf * 8
    # bytes the three kernels move in this design (K_e round trip through HBM)
    n_contrib = 16 * ne
    moved = alg + ne * (144 + 12) * 8 * 2 + n_contrib * 4 + info["node_pairs"] * 24
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks["hbm_gbs"])  # measured copy bandwidth (driver-written)
    achieved = alg / (ms * 1e-3) / 1e9
    # CPU baseline: oracle C restatement, one thread, bounded mesh
    import oracle as O
    cm, cn, cr = make_case(args.cpu_cells, 2)
    t = time.perf_counter()
    O.assemble(cm.tets, cm.coords.ravel(), cr[:, :6], cr[:, 6:], cn.free_of_dof, cn.n_free)
    cpu_s = time.perf_counter() - t
    line = {
        "metric": "macro assembly tets/s (residual + free x free stiffness, bitwise "
                  "macrofem.cpp:104-187)",
        "value": ne / (ms * 1e-3), "unit": "tets/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"box mesh {args.cells}^3 cells ({ne} tets, {mesh.n_nodes} "
                               f"nodes, n_free {nf}, nnz {nnz}), random sigma/C records",
                   "l2": "flushed between timed steps (256 MiB device write)",
                   "plan_build_s": round(plan_s, 3)},
        "kernel_ms": {"element": parts[0], "pair_gather": parts[1], "residual": parts[2]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": None,
                     "alg_bytes_per_step": alg, "design_bytes_per_step": moved,
                     "design_gbps": moved / (ms * 1e-3) / 1e9},
        "gpu_launches": 3 * args.steps,
        "e2e": {"value": ne / (e2e_ms * 1e-3), "unit": "tets/s",
                "h2d_bytes_per_step": mesh.n_nodes * 24 + ne * 42 * 8,
                "d2h_bytes_per_step": (nf + nnz) * 8},
        "cpu_baseline": {"value": cm.n_elements / cpu_s, "unit": "tets/s", "cores": 1,
                         "kind": "port", "sample": f"oracle or_assemble on a {args.cpu_cells}^3 "
                         f"box ({cm.n_elements} tets, {cpu_s:.2f} s)"},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
