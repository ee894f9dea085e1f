#!/usr/bin/env python
"""Benchmark: DG Euler RHS + LSERK4 stage throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

A "step" is one LSERK4 time step = 5 RK stages, each one fused sm_100a stage
kernel (volume flux, face flux + LIFT, DMMA contraction, LSERK update) over the
whole mesh.  value = DOFs x stages / time  in GDOF/s per RK stage (DOF = K Np 5,
DESIGN.md A15), whole job over all ranks (max-over-ranks device time).

Default workload: C4 (BASELINE.json configs[3]: 1.47M affine tets, N = 4, horn
cavity with slip walls, pass-through outer boundary, 10 % pulse) -- the config
the metric's 1/2/4/8-GPU scaling and its "largest mesh" target are stated on
(DESIGN.md "Measurement").  N > 1: launched by torchrun, x-slab element
partition, NCCL face-trace halo every stage (strong scaling).

--impl reference: the CPU oracle (oracle/, plain numpy fp64) timed as it stands
on this host's cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DG Euler RHS+RK stage GDOF/s at 1/2/4/8 B200; % of HBM/FP64 roofline"
UNIT = "GDOF/s"
FP64_PEAK_TFLOPS = 37.04      # measured: DMMA m16n8k16 microbenchmark, profiles/r01_fp64_peak.txt
STAGES = 5


def flops_per_elem_stage(N: int) -> float:
    """Algorithmic FLOPs per element per RK stage."""
    Np = (N + 1) * (N + 2) * (N + 3) // 6
    Nfp = (N + 1) * (N + 2) // 2
    return 30 * Np ** 2 + 40 * Np * Nfp + 110 * Np + 480 * Nfp + 25 * Np


def flops_per_elem_stage_modal(p: int) -> float:
    """Algorithmic FLOPs per element per stage of the modal-quadrature scheme (A23):
    interpolation to NQ = (p+1)^3 volume and 4 NQF = 4 (p+1)^2 face points (own and neighbour),
    fluxes there, weak-form projections back onto Np modes, the update."""
    Np = (p + 1) * (p + 2) * (p + 3) // 6
    NQ, NQF = (p + 1) ** 3, (p + 1) ** 2
    return (2 * NQ * Np * 5 + 110 * NQ + 2 * 3 * NQ * Np * 5          # volume
            + 2 * 2 * 4 * NQF * Np * 5 + 120 * 4 * NQF + 2 * 4 * NQF * Np * 5 + 25 * Np)   # faces, update


def bytes_per_elem_stage(N: int) -> float:
    """Compulsory HBM bytes per element per stage: Q and res read+written + geometry + connectivity."""
    Np = (N + 1) * (N + 2) * (N + 3) // 6
    return 4 * 5 * Np * 8 + 200 + 24


def roofline(fpe, bpe, K_loc, per_launch_ms, traffic):
    """The roofline that binds the stage kernel (max of compulsory bytes / HBM_BW and
    algorithmic flops / FP64_peak): FP64 ("tensor": the DMMA and DFMA pipes share one measured rate)
    from N = 3 up, HBM at N <= 2 (N = 1: 3.4 flop/B against a ridge of 5.7).  Both fractions are
    always reported."""
    hbm_peak = measured_peaks().get("hbm_gbs", 6545.0)
    sec = per_launch_ms * 1e-3
    tf = fpe * K_loc / sec / 1e12
    gbs = bpe * K_loc / sec / 1e9
    f_frac, h_frac = tf / FP64_PEAK_TFLOPS, gbs / hbm_peak
    common = {"traffic": traffic, "flops_per_elem_stage": fpe, "hbm_bytes_per_elem_stage": bpe,
              "fp64_frac": round(f_frac, 4), "hbm_frac": round(h_frac, 4),
              "peak_source": "FP64: measured DMMA peak %.2f TFLOP/s (profiles/r01_fp64_peak.txt; MEASURED_PEAKS.json "
                             "has no FP64); HBM: MEASURED_PEAKS.json hbm_gbs (else 6545)" % FP64_PEAK_TFLOPS}
    if bpe / (hbm_peak * 1e9) > fpe / (FP64_PEAK_TFLOPS * 1e12):
        return {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(h_frac, 4), **common}
    return {"bound": "tensor", "achieved": round(tf, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": round(f_frac, 4), **common}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        rows = [r.split(",") for r in (self.out or "").strip().splitlines() if r.strip()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 5 + i and "Active" in r[5 + i]
                          and "Not" not in r[5 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def build_config(name: str, nparts: int):
    from synth import configs
    if name == "C5":
        return configs.make("C5", nparts=nparts)
    return configs.make(name)


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1710_03887_b200 as dg
    from synth import configs, mesh as smesh

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = build_config(args.config, world)
    if args.order:
        cfg.order = args.order
    modal = args.scheme == "modal"
    m = cfg.mesh
    part = smesh.x_slab_partition(m, world) if world > 1 else None
    s = dg.Solver(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma, q_inf=cfg.q_inf,
                  part=part, nparts=world, rank=rank,
                  scheme=dg.DG_SCHEME_MODAL if modal else dg.DG_SCHEME_NODAL)
    if world > 1:
        uid = [dg.dg_nccl_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        dg.dg_comm_init(s.ctx, uid[0], world)
    if args.reserve_sms:
        # leave SMs free for the NCCL halo kernels so they overlap the interior launch
        s.set_max_ctas(torch.cuda.get_device_properties(dev).multi_processor_count - args.reserve_sms)
    x = s.nodes()
    Q0 = configs.initial_state(cfg, x)                  # synthetic state at the library's nodes
    s.set_state(Q0)
    dt = s.stable_dt(cfg.cfl)
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        dt = float(t.item())
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    # ---------------- device-resident throughput
    s.step(dt, args.warmup)
    barrier()
    n0 = dg.dg_launch_count(s.ctx)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        s.step(dt, args.steps)
        e1.record(stream)
        barrier()
        launches = dg.dg_launch_count(s.ctx) - n0
        ms = e0.elapsed_time(e1)
        # nvidia-smi samples every 200 ms: a timed region shorter than ~1 s is followed, inside
        # the sampling window, by untimed repeats of the same steps so the clocks are read under
        # this workload (same count on every rank: the steps exchange halos)
        reps = min(2000, int(1000.0 / max(ms, 1e-3)) + 1) if ms < 1000.0 else 0
        if world > 1:
            r = torch.tensor([reps], dtype=torch.int64, device=dev)
            dist.all_reduce(r, op=dist.ReduceOp.MAX)
            reps = int(r.item())
        for _ in range(reps):
            s.step(dt, args.steps)
        barrier()
    clk_info = clk.summary()
    if reps:
        clk_info["window"] = f"timed region + {reps * args.steps} untimed steps of the same workload"
    dg.dg_check(s.ctx, s.stream)
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    K_tot = m.K
    dofs = K_tot * s.Np * 5
    ranks_info = None
    if world > 1:
        # per-rank evidence for the scaling run: own stage time, halo size, halo-only time
        nh = max(1, args.steps)
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        h0.record(stream)
        for _ in range(nh):
            dg.dg_halo_exchange(s.ctx, s.stream)
        h1.record(stream)
        barrier()
        npeer, nsend, nrecv = dg.dg_halo_info(s.ctx)
        mine = {"rank": rank, "elements": int(s.K), "ms_steps": round(ms, 4),
                "ms_per_stage": round(ms / (STAGES * args.steps), 5), "peers": npeer,
                "halo_send_bytes_per_stage": int(nsend * 5 * s.Nfp * 8),
                "halo_recv_bytes_per_stage": int(nrecv * 5 * s.Nfp * 8),
                "halo_only_ms_per_exchange": round(h0.elapsed_time(h1) / nh, 5)}
        ranks_info = [None] * world
        dist.all_gather_object(ranks_info, mine)
    value = dofs * STAGES * args.steps / (ms_max * 1e-3) / 1e9

    # ---------------- stage-kernel timing on its own stream (roofline numerator)
    per_launch_ms = ms / (STAGES * args.steps) if launches else None
    # single-rank stage kernels only: with P > 1 a stage is two launches (interior, boundary)
    if world > 1 and per_launch_ms is not None:
        per_launch_ms = ms / (STAGES * args.steps)
    K_loc = s.K
    fpe = flops_per_elem_stage_modal(cfg.order) if modal else flops_per_elem_stage(cfg.order)
    flops_launch = fpe * K_loc
    traffic = None
    # committed ncu summary of this kernel on this workload: the BASELINE configs, or the C4 mesh at
    # an overridden order / in the modal scheme (ncu_summary_C4_N1.json, ncu_summary_C4_modal1.json)
    tag = args.config if not (modal or args.order) else f"{args.config}_{'modal' if modal else 'N'}{cfg.order}"
    prof = os.path.join(ROOT, "profiles", f"ncu_summary_{tag}.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---------------- end to end through the public API with host buffers
    Qh = torch.from_numpy(np.ascontiguousarray(Q0)).pin_memory()
    Qo = torch.empty_like(Qh).pin_memory()
    inp = [Qh[i].data_ptr() for i in range(5)]
    outp = [Qo[i].data_ptr() for i in range(5)]
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    t0 = time.perf_counter()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(e2e_steps):
        dg.dg_set_state(s.ctx, inp, False, 0.0, s.stream)
        dg.dg_rk_step(s.ctx, dt, 1, s.stream)
        dg.dg_get_state(s.ctx, outp, False, s.stream)
    f1.record(stream)
    barrier()
    e2e_ms = f0.elapsed_time(f1)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = dofs * STAGES * e2e_steps / (e2e_ms * 1e-3) / 1e9
    state_bytes = 5 * K_loc * s.Np * 8

    if rank == 0:
        cpu = cpu_baseline(args, cfg) if (world == 1 and not args.no_cpu_baseline and not modal) else None
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
            "scaling": "weak" if args.config == "C5" else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded mesh + isentropic Gaussian pulse, DESIGN.md input recipe)",
            "config": {"workload": f"{args.config}{' modal-quadrature scheme' if modal else ''}: K={K_tot} affine tets, N={cfg.order}, Np={s.Np}, "
                                   f"{len(cfg.pulses)} pulse(s), LSERK4 dt={dt:.4g} (CFL {cfg.cfl})",
                       "elements": K_tot, "order": cfg.order, "dofs": dofs, "stages_per_step": STAGES,
                       "parallelism": f"x-slab element partition x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (state %.2f GB vs 126 MB L2)" % (5 * K_tot * s.Np * 8 / 1e9)},
            "roofline": roofline(fpe, bytes_per_elem_stage(cfg.order), K_loc, per_launch_ms, traffic),
            "clocks": clk_info,
            "e2e": {"value": round(e2e_value, 4), "unit": UNIT, "h2d_bytes_per_step": state_bytes,
                    "d2h_bytes_per_step": state_bytes, "steps": e2e_steps,
                    "api": "dg_set_state(host pinned) + dg_rk_step(1) + dg_get_state(host pinned)"},
            "gpu_launches": int(launches),
            "cpu_baseline": cpu,
            "build": build_info(dg),
        }
        if ranks_info is not None:
            line["ranks"] = ranks_info
        if args.reserve_sms:
            line["config"]["reserve_sms"] = args.reserve_sms
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def build_info(dg):
    try:
        return dg.dg_build_info()
    except AttributeError:          # an older library build without the call
        return None


# ------------------------------------------------------------------ oracle (CPU)
def _oracle_sample_step(cfg, nsample):
    """One LSERK4 stage of the oracle over `nsample` contiguous elements of the workload."""
    from oracle import timestep
    from oracle.rhs import OracleMesh, rhs
    from synth import configs
    m = cfg.mesh
    o = OracleMesh(order=cfg.order, vxyz=m.vxyz, etov=m.etov, bc=m.bc, etoe=m.etoe, etof=m.etof,
                   gamma=cfg.gamma, q_inf=cfg.q_inf)
    lo = max(0, m.K // 2 - nsample // 2)
    elems = np.arange(lo, lo + nsample)
    patch = np.unique(np.concatenate([elems, m.etoe[elems].ravel()]))
    from oracle import geom
    xp = geom.node_coordinates(m.vxyz, m.etov[patch], o.ref.r, o.ref.s, o.ref.t)
    Q = np.zeros((5, m.K, o.Np))
    Q[:, patch] = configs.initial_state(cfg, xp)
    res = np.zeros((5, nsample, o.Np))
    a, b = timestep.LSERK4_A[1], timestep.LSERK4_B[1]
    o.vmaps(elems)                                    # connectivity set-up outside the timing

    def stage():
        k = rhs(o, Q, 0.0, elems=elems)
        r = a * res + 1e-3 * k
        return Q[:, elems] + b * r

    return o, stage


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        n = max((i.get("num_threads", 0) for i in threadpool_info()), default=0)
        return int(n) or os.cpu_count()
    except Exception:
        return os.cpu_count()


def _cpu_seconds():
    r = os.times()
    return r.user + r.system


def cpu_baseline(args, cfg, budget_s=12.0):
    nsample = 4096 if cfg.order >= 5 else 16384
    o, stage = _oracle_sample_step(cfg, nsample)
    stage()                                            # warm
    t0 = time.perf_counter()
    c0 = _cpu_seconds()
    n = 0
    while time.perf_counter() - t0 < budget_s or n == 0:
        stage()
        n += 1
    wall = time.perf_counter() - t0
    dt = wall / n
    value = nsample * o.Np * 5 / dt / 1e9
    # cores actually used: process CPU time / wall time (numpy's elementwise work is
    # single-threaded; only the matrix products use the BLAS threads)
    used = (_cpu_seconds() - c0) / wall
    return {"value": round(value, 6), "unit": UNIT, "cores": round(used, 2), "kind": "oracle",
            "blas_threads": cpu_cores(), "host_cpus": os.cpu_count(),
            "sample": f"{n} oracle LSERK4 stages (rhs + update) over {nsample} contiguous elements of {args.config}, "
                      f"{dt:.3f} s/stage"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = build_config(args.config, 1)
    nsample = 2048 if cfg.order >= 5 else 8192
    o, stage = _oracle_sample_step(cfg, nsample)
    for _ in range(args.warmup):
        stage()
    t0 = time.perf_counter()
    c0 = _cpu_seconds()
    for _ in range(args.steps):
        stage()
    wall = time.perf_counter() - t0
    used = (_cpu_seconds() - c0) / wall
    dt = wall / args.steps
    value = nsample * o.Np * 5 / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "weak" if args.config == "C5" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded)",
        "config": {"workload": f"{args.config} (oracle sample of {nsample} elements, one RK stage per step)",
                   "elements": int(cfg.mesh.K), "order": cfg.order},
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "kind": "oracle", "cores": round(used, 2),
                         "blas_threads": cpu_cores(), "host_cpus": os.cpu_count(),
                         "sample": f"{nsample} contiguous elements of {args.config}, 1 LSERK4 stage per step"},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scheme", default="nodal", choices=["nodal", "modal"],
                    help="modal = the paper's modal-quadrature scheme (orders 1-3; SURVEY N3)")
    ap.add_argument("--order", type=int, default=0, help="override the config's polynomial order")
    ap.add_argument("--reserve-sms", type=int, default=0,
                    help="stage-kernel grid = SMs - k (leave SMs to the NCCL halo kernels, N > 1)")
    args = ap.parse_args()
    # run-time experiment switches would change what is timed: refuse them (the build's own
    # compile-time configuration is recorded in the JSON line as "build")
    dg_env = sorted(k for k in os.environ if k.startswith("DG_"))
    if dg_env:
        raise SystemExit(f"bench.py refuses to run with DG_* experiment variables set: {dg_env}")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched without torchrun: spawn the N ranks ourselves (one process per GPU, NCCL);
        # rank 0 prints the JSON line
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
