#!/usr/bin/env python
"""Benchmark of the B200 batched RVE solver (BASELINE.json metric, config 2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--tangent]
                  [--config 2|3|4|5]

Default (the headline, BASELINE configs[1]): a step = one batch_response over one shard of
synthetic RVEs: 1,024 same-topology
~1k-fiber knn RVEs (375 nodes / 1000 fibers, seed 1 = the config-1 network) with distinct
deformation gradients (mt19937_64(55) recipe of test_batch.cpp:149-157), each relaxed to
convergence by DR followed by homogenized stress ("stress only", BASELINE configs[1]).
With --tangent every point also runs the 6 warm-started probes and the tangent (config 5).
Under torchrun each rank solves its own 1,024 points (weak scaling) and the result
records are gathered with one NCCL all-gather.
--config 3|4|5 (strong scaling, the fixed batch is cut into fiber-weighted
contiguous shards): 3 = 16,384 heterogeneous knn RVEs of 500-5k fibers (one network per
point), 4 = 64 jittered-lattice RVEs of 50k fibers (16-CTA clusters), 5 = the first 4,096
config-3 RVEs with base + 6 probes + tangent.

Headline line (rank 0, one JSON line):
  value    RVE-solves/s over all ranks with F resident in HBM (device-timed, CUDA events,
           max over ranks, L2 flushed between steps)
  e2e      same metric through the public batch_response with host PackedStates
           (H2D of F + warm states, D2H of results + states inside the timed region)
  roofline FP64-pipe ops of the DR kernel / its event time vs the FP64 pipe peak measured
           on this device (fibra_cuda_fp64_peak)
  cpu_baseline  the reference's own compiled DR (oracle/_ref) on the host cores, bounded
           sample of the same workload; "single_rve" = the 1-core, best-of-3 config-1 rate
           at lambda = 1.05 and 1.25 (the >= 1000x denominator).
--impl reference times only that CPU implementation (all host threads) and prints the same
metric line with "impl": "reference" and the same "config".  It imports nothing from the
product package: the network comes from the reference's own generator (oracle/_ref) and F
from oracle/workload.py; its timed steps together solve every point of the config-2 batch.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RVE solves/s (DR to convergence + homogenized stress), config 2"
METRICS = {2: METRIC,
           3: "RVE solves/s (DR to convergence + homogenized stress), config 3",
           4: "RVE solves/s (DR to convergence + homogenized stress), config 4",
           5: "RVE responses/s (base + 6 probes, stress + tangent), config 5"}
DEFAULT_POINTS = {2: 1024, 3: 16384, 4: 64, 5: 4096}
UNIT = "RVE-solves/s"
POINTS = 1024
NET_SEED = 1


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5])
    ap.add_argument("--points", type=int, default=None,
                    help="config 2: points per GPU; configs 3-5: points in the whole batch")
    ap.add_argument("--tangent", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--single-process", action="store_true",
                    help="one process drives all --gpus through the library's multi-device "
                         "context (fibra_cuda_open_devices: LPT shards, one ncclAllGather); "
                         "run without torchrun")
    a = ap.parse_args()
    if a.points is None:
        a.points = DEFAULT_POINTS[a.config]
    if a.config == 5:
        a.tangent = True
    return a


def proxy_cost(m, n):
    """The library's schedule cost model without the network-specific degree term (computable
    from the config-3 recipe alone, so every rank plans without building all networks)."""
    return np.exp(-3.3 * m / n + 1.75 * np.log(m)) * m


def workload(args, world, rank, full=False):
    """(networks, entry_of_point, F (n, 9), description, global point count, scaling) of
    this rank's shard (``full``: the whole batch of all ``world`` GPUs, for one process).
    Configs 3-5 shard by longest-processing-time on the cost model (shard.plan_shards)."""
    import paper_2306_09427_b200 as P
    from paper_2306_09427_b200 import synth
    from paper_2306_09427_b200.shard import plan_shards
    tangent = args.tangent
    if args.config == 2:
        points = args.points
        net = P.generate_network(synth.config1_spec(), NET_SEED)
        F_all = synth.batch_F(points * world)
        if full:
            F = np.ascontiguousarray(F_all).reshape(points * world, 9)
            desc = describe(args, world, points, points * world, "weak", net.n_free)[0]
            return [net], np.zeros(points * world, np.int32), F, desc, points * world, "weak"
        F = np.ascontiguousarray(F_all[rank * points:(rank + 1) * points]).reshape(points, 9)
        desc = (f"config{5 if tangent else 2}: {points} same-topology knn RVEs per GPU "
                f"(375 nodes/1000 fibers, seed {NET_SEED}, n_free {net.n_free}), distinct F "
                f"(mt19937_64(55) recipe), {'base + 6 probes + tangent' if tangent else 'stress only'}")
        return [net], np.zeros(points, np.int32), F, desc, points * world, "weak"
    total = args.points
    if args.config == 4:
        cost = np.full(total, 50000.0)
        make = synth.config4_network
    else:
        mn = np.array([synth.config3_size(p) for p in range(total)], dtype=np.float64)
        cost = proxy_cost(mn[:, 0], mn[:, 1])
        make = synth.config3_network
    pts = np.arange(total) if full else plan_shards(cost, world)[rank]
    nets = synth.parallel_networks(make, [int(p) for p in pts])
    F = np.ascontiguousarray(synth.batch_F(total)[pts]).reshape(len(pts), 9)
    kind = {3: "heterogeneous knn RVEs of 500-5k fibers (SURVEY 8d recipe, one network per point)",
            4: "jittered-lattice RVEs of 50k fibers / 12,167 nodes (16-CTA clusters)",
            5: "config-3 RVEs (first 4,096), base + 6 warm probes + tangent"}[args.config]
    desc = (f"config{args.config}: {total} {kind}, distinct F (mt19937_64(55) recipe), "
            f"longest-processing-time shards on the cost model")
    return nets, np.arange(len(pts), dtype=np.int32), F, desc, total, "strong"


def describe(args, world, n_per_gpu, total, scaling, n_free):
    """Workload description and the `config` dict, shared verbatim by both arms."""
    if args.config == 2:
        desc = (f"config{5 if args.tangent else 2}: {n_per_gpu} same-topology knn RVEs per GPU "
                f"(375 nodes/1000 fibers, seed {NET_SEED}, n_free {n_free}), distinct F "
                f"(mt19937_64(55) recipe), "
                f"{'base + 6 probes + tangent' if args.tangent else 'stress only'}")
    else:
        kind = {3: "heterogeneous knn RVEs of 500-5k fibers (SURVEY 8d recipe, one network per point)",
                4: "jittered-lattice RVEs of 50k fibers / 12,167 nodes (16-CTA clusters)",
                5: "config-3 RVEs (first 4,096), base + 6 warm probes + tangent"}[args.config]
        desc = (f"config{args.config}: {total} {kind}, distinct F (mt19937_64(55) recipe), "
                f"longest-processing-time shards on the cost model")
    cfg = {"workload": desc, "points_per_gpu": n_per_gpu, "global_points": total,
           "l2": "flushed between timed steps (256 MiB device write)",
           "parallelism": f"dp{world} (independent RVE shards, 1 NCCL all-gather "
                          "of result records per step)"}
    return desc, cfg


def sample_points(n, sample):
    """Bounded CPU sample: evenly spaced points of the shard (all of them when small)."""
    return np.unique(np.linspace(0, n - 1, min(n, sample)).astype(int))


def step_slices(n, steps, min_size):
    """Point slices of the CPU reference run: a fixed interleaving permutation of the n points
    (stride coprime with n, so every slice mixes cheap and capped solves), cut into `steps`
    consecutive slices of max(ceil(n / steps), min_size) points, wrapping around: over the
    timed steps every point of the batch is solved at least once."""
    stride = next(s for s in range(int(n * 0.618) | 1, 2 * n + 2) if np.gcd(s, n) == 1)
    perm = (np.arange(n) * stride) % n
    size = max(-(-n // steps), min(min_size, n))
    return [perm[(k * size + np.arange(size)) % n] for k in range(steps)]


def single_rve_baseline():
    """BASELINE.md 4.2 denominator: the reference's relax_solve + homogenized_stress
    (oracle/_ref, relax.cpp:93-191, network.cpp:341-372) on ONE core, best of 3, for the
    config-1 network (knn 375/1000, seed 1) at F = diag(lambda, 1, 1), lambda = 1.05 and 1.25."""
    import oracle as O
    from oracle import workload as W
    if not O.ref_available():
        return None
    rnet = O.ref_generate(seed=W.NET_SEED, **W.CONFIG1_KNN)
    out = {"cores": 1, "kind": "reference", "network": "knn 375 nodes/1000 fibers seed 1",
           "repeats": "best of 3"}
    for lam in (1.05, 1.25):
        F = np.diag([lam, 1.0, 1.0])
        best, its = float("inf"), 0
        for _ in range(3):
            t0 = time.perf_counter()
            st, rep = O.ref_relax_solve(rnet, F)
            O.ref_homogenized_stress(rnet, st, F)
            best = min(best, time.perf_counter() - t0)
            its = rep["iterations"]
        out[f"lambda_{lam}"] = {"solves_per_s": 1.0 / best, "seconds": best, "iterations": its,
                                "ns_per_fiber_iteration": best / (its * rnet.n_fibers) * 1e9}
    return out


def cpu_sample_rate(args, nets, eop, F, n_workers, sample):
    """Reference CPU implementation on the host cores over a bounded sample of the workload:
    oracle/_ref (the reference's own translation units) for the headline config 2, else the
    oracle restatement.  Returns (rve_solves_per_s, kind, seconds, iterations, n_sampled)."""
    import oracle as O
    from oracle import workload as W
    idx = sample_points(len(F), sample)  # evenly spaced: iteration counts are heavy-tailed
    if args.config == 2 and O.ref_available() and not args.tangent:
        rnet = O.ref_generate(seed=W.NET_SEED, **W.CONFIG1_KNN)
        t0 = time.perf_counter()
        sig, iters, status = O.ref_batch_stress(rnet, F[idx], workers=n_workers)
        dt = time.perf_counter() - t0
        return len(idx) / dt, "reference", dt, int(iters.sum()), len(idx)
    O.build(ref=False)
    used = sorted({int(eop[i]) for i in idx})
    remap = {e: k for k, e in enumerate(used)}
    onets = [O.Network(nets[e].coords, nets[e].fiber_nodes[:, 0], nets[e].fiber_nodes[:, 1],
                       nets[e].fiber_area, nets[e].fiber_modulus, nets[e].box_half) for e in used]
    seop = [remap[int(eop[i])] for i in idx]
    st = O.PackedStates.fresh(onets, seop)
    t0 = time.perf_counter()
    resp, status = O.batch_response(onets, seop, st, F[idx], want_tangent=args.tangent,
                                    n_threads=n_workers)
    dt = time.perf_counter() - t0
    return len(idx) / dt, "port", dt, int(sum(r["relax_iterations"] for r in resp)), len(idx)


def run_reference(args, rank, world):
    """The reference's own CPU implementation of the path on this box's host cores.

    Config 2 (the headline): the network comes from the reference's own generator and every
    DR solve from the reference's compiled relax_solve / homogenized_stress (oracle/_ref,
    WorkerPool over all host threads); the F recipe from oracle/workload.py.  Nothing of the
    product package is imported.  The timed steps together cover the whole config-2 batch
    of GPU shard 0 (1,024 points), so the rate is over the same points the GPU arm solves.
    Configs 3-5 (builder runs only) time the oracle port on the product's networks."""
    if rank != 0:
        return
    import oracle as O
    from oracle import workload as W
    n_workers = os.cpu_count() or 1
    if args.config == 2 and O.ref_available() and not args.tangent:
        rnet = O.ref_generate(seed=W.NET_SEED, **W.CONFIG1_KNN)
        n = args.points
        F = np.ascontiguousarray(W.batch_F(n * world)[:n]).reshape(n, 9)
        desc, cfg = describe(args, world, n, n * world, "weak", rnet.n_free)
        scaling = "weak"
        slices = step_slices(n, args.steps, 2 * n_workers)
        if args.warmup > 0:
            O.ref_batch_stress(rnet, F[slices[0][:n_workers]], workers=n_workers)
        secs, iters, done, covered = 0.0, 0, 0, set()
        for sl in slices:
            t0 = time.perf_counter()
            _, its, _ = O.ref_batch_stress(rnet, F[sl], workers=n_workers)
            secs += time.perf_counter() - t0
            iters += int(its.sum())
            done += len(sl)
            covered.update(int(p) for p in sl)
        kind = "reference"
        assert "paper_2306_09427_b200" not in sys.modules  # reference arm: no product code
        sample = (f"all {len(covered)} of {n} points of GPU shard 0 across the {args.steps} "
                  f"timed steps ({done // args.steps} interleaved points per step), "
                  f"{n_workers} WorkerPool threads")
    else:
        import paper_2306_09427_b200  # noqa: F401  (configs 3-5: the product's host generator)
        nets, eop, F, _, total, scaling = workload(args, 1, 0)
        desc, cfg = describe(args, world, len(F), total, scaling, None)
        sample = max(8, 4 * n_workers)
        secs, iters, done = 0.0, 0, 0
        kind = "port"
        for _ in range(args.steps):
            r, kind, dt, its, k = cpu_sample_rate(args, nets, eop, F, n_workers, sample)
            secs += dt
            iters += its
            done += k
        sample = (f"evenly spaced {done // args.steps} points of the workload per step, "
                  f"{n_workers} threads")
    value = done / secs
    line = {"impl": "reference", "metric": METRICS[args.config], "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "dr_iter_rve_per_s": iters / secs,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": n_workers, "kind": kind,
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if args.config == 2 and not args.no_cpu_baseline:
        line["cpu_baseline"]["single_rve"] = single_rve_baseline()
    print(json.dumps(line), flush=True)


def measured_capture(args):
    """The committed ncu --set full capture of this exact workload's DR launch
    (profiles/r02_dr_traffic.json), else None."""
    path = os.path.join(ROOT, "profiles", "r02_dr_traffic.json")
    if args.config != 2 or args.tangent or args.points != DEFAULT_POINTS[2] or not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)


def measured_traffic(args, n_steps):
    """DRAM bytes per DR launch from the committed capture, else None."""
    cap = measured_capture(args)
    return cap["dram_bytes_per_launch"] if cap else None


def measured_smem(args):
    """Shared-memory pipe figures of the DR kernel from the committed capture, else None."""
    cap = measured_capture(args)
    if not cap or "smem_wavefronts_per_launch" not in cap:
        return None
    return {"wavefronts_per_rve_iteration": cap["smem_wavefronts_per_launch"] / cap["rve_iterations_per_launch"],
            "pipe_pct_of_peak": cap["smem_pipe_pct_of_peak_elapsed"],
            "source": "ncu --set full of one config-2 DR launch (profiles/r02_dr_traffic.json)"}


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2306_09427_b200 as P

    sp = args.single_process and args.gpus > 1  # one process, the library's multi-device path
    devices = list(range(args.gpus)) if sp else None
    ngpu = args.gpus if sp else world
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if sp:
        nets, eop, F, desc, total, scaling = workload(args, args.gpus, 0, full=True)
    else:
        nets, eop, F, desc, total, scaling = workload(args, world, rank)
    n = len(F)
    lib = P.RveLibrary(nets, policy="explicit", explicit_assignment=[int(e) for e in eop])
    assign = P.BatchAssignment(eop)
    stream = torch.cuda.Stream(device=local)  # explicit stream shared by torch and the solver
    torch.cuda.set_stream(stream)
    if sp:
        db = P.DeviceBatch(lib, assign, device=0, devices=devices)
    else:
        db = P.DeviceBatch(lib, assign, device=local, stream=stream.cuda_stream)
    peak = db.fp64_peak()  # FP64-pipe roofline denominator, measured while the GPU is idle
    rec_bytes = P.RESULT_DTYPE.itemsize
    F_dev = torch.from_numpy(F).to(f"cuda:{local}")
    # the all-gather moves equal-size buffers: shards are padded to the largest one
    counts = torch.tensor([n], dtype=torch.int64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.MAX)
    n_pad = int(counts.item())
    out_dev = torch.zeros(n_pad * rec_bytes, dtype=torch.uint8, device=f"cuda:{local}")
    gathered = torch.empty(world * n_pad * rec_bytes, dtype=torch.uint8, device=f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")
    law, rcfg, scfg = P.FiberLaw(), P.RelaxConfig(), P.StiffnessConfig()

    def step():
        db.solve_device(F_dev.data_ptr(), out_dev.data_ptr(), law, rcfg, scfg, args.tangent)
        if world > 1:
            dist.all_gather_into_tensor(gathered, out_dev)

    for _ in range(args.warmup):
        db.reset_states()
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    total_ms, dr_ms, iters, pipe_ops, fiber_iters, failed, launches = 0.0, 0.0, 0, 0, 0, 0, 0
    alg_flops = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.start()
    for _ in range(args.steps):
        flush.fill_(1)  # L2 flush between timed steps (256 MiB > 126 MB L2)
        db.reset_states()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        step()
        ev1.record(stream)
        torch.cuda.synchronize()
        s = db.last_stats()
        if sp:  # the devices run on the library's streams: its events on device 0 span the
            db.synchronize()  # F gather, every device's solve, the all-gather and the permute
            total_ms += s["total_ms"]
        else:
            total_ms += ev0.elapsed_time(ev1)
        dr_ms += s["dr_kernel_ms"]
        iters += s["iterations"]
        pipe_ops += s["pipe_ops"]
        fiber_iters += s["fiber_iterations"]
        launches += s["kernel_launches"]
        alg_flops += s["alg_flops"]
    clk = clocks.stop()
    rec = np.frombuffer(out_dev.cpu().numpy().tobytes(), dtype=P.RESULT_DTYPE)[:n]
    failed_t = torch.tensor([int((rec["status"] != 0).sum())], device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(failed_t)
    failed = int(failed_t.item())

    t = torch.tensor([total_ms, dr_ms], dtype=torch.float64, device=f"cuda:{local}")
    tot_iters = torch.tensor([iters, pipe_ops, fiber_iters, alg_flops], dtype=torch.float64,
                             device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot_iters, op=dist.ReduceOp.SUM)
    max_total_ms, max_dr_ms = t.tolist()
    all_iters, all_pipe, all_fib, all_flops = tot_iters.tolist()
    value = total * args.steps / (max_total_ms * 1e-3)

    # ---- end to end through the public API with host buffers ----
    st_host, _ = P.init_batch(np.zeros(n, np.int32), lib, 0)  # explicit policy -> eop
    st_host.offsets = st_host.offsets  # fresh zero-filled PackedStates (init_batch)
    e2e_s = 0.0
    for i in range(args.e2e_steps + 1):
        for k in ("u", "t", "iters", "converged"):
            getattr(st_host, k)[:] = 0
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        br = P.batch_response(lib, assign, st_host, law, F, rcfg, scfg,
                              want_tangent=args.tangent, device=local, devices=devices)
        if world > 1:
            g = torch.zeros(n_pad * rec_bytes, dtype=torch.uint8, device=f"cuda:{local}")
            g[:n * rec_bytes] = torch.from_numpy(br.records.view(np.uint8).copy()).to(f"cuda:{local}")
            dist.all_gather_into_tensor(gathered, g)
            torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i > 0:  # first call includes context creation
            e2e_s += dt
    et = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_val = total * args.e2e_steps / et.item()
    tot = int(st_host.total_dofs())
    h2d = n * 72 + tot * 8 + n * (8 + 8 + 1)
    d2h = n * rec_bytes + 7 * tot * 8 + n * (8 + 8 + 1)

    if rank == 0:
        achieved = all_pipe / ngpu / (max_dr_ms * 1e-3)  # per-GPU FP64-pipe lane-ops/s
        cfg = describe(args, ngpu, n // ngpu if sp and args.config == 2 else n, total, scaling,
                       nets[0].n_free if args.config == 2 else None)[1]
        if sp:
            cfg["parallelism"] = (f"dp{ngpu} in one process (fibra_cuda_open_devices: "
                                  "longest-processing-time shards, 1 ncclAllGather of the "
                                  "result records per step)")
        line = {
            "metric": METRICS[args.config], "value": value, "unit": UNIT, "n_gpus": ngpu,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": max_total_ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "dr_iter_rve_per_s": all_iters / (max_total_ms * 1e-3) * (args.steps / args.steps),
            "failed_points": failed,
            "roofline": {"bound": "fp64_pipe", "achieved": achieved / 1e9, "peak": peak / 1e9,
                         "unit": "Gop/s (FP64-pipe lane ops)", "frac": achieved / peak,
                         "traffic": measured_traffic(args, args.steps),
                         "traffic_unit": "DRAM bytes per DR launch (ncu --set full, profiles/r02_dr_traffic.json)",
                         "shared_memory": measured_smem(args),
                         "work_model": "W_pipe = 51 M + 12 n_free + 2 n_fix per RVE-iteration "
                                       "(SURVEY 8d); peak measured by a DADD stream on this "
                                       "device"},
            "alg_flops": {"achieved_tflops": all_flops / ngpu / (max_dr_ms * 1e-3) / 1e12,
                          "fma_peak_tflops": 2 * peak / 1e12,
                          "frac": all_flops / ngpu / (max_dr_ms * 1e-3) / (2 * peak),
                          "model": "F_alg = 28 M + 12 n_free + 2 n_fix flops per RVE-iteration "
                                   "(div and sqrt count 1; SURVEY 8d); peak = 2 x the measured "
                                   "DADD lane-op rate (FMA-counted)"},
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
        }
        if world == 1 and not args.no_cpu_baseline:
            nw = os.cpu_count() or 1
            sample = max(8, 4 * nw)  # >> threads: the heavy tail must not idle the pool
            r, kind, secs, its, k = cpu_sample_rate(args, nets, eop, F, nw, sample)
            which = "evenly spaced"
            line["cpu_baseline"] = {"value": r, "unit": UNIT, "cores": nw, "kind": kind,
                                    "sample": f"{which} {k} points of this workload on "
                                              f"{nw} host threads ({secs:.1f} s, {its} DR "
                                              "iterations)"}
            single = single_rve_baseline()
            if single is not None:
                line["cpu_baseline"]["single_rve"] = single
        print(json.dumps(line), flush=True)
    db.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
