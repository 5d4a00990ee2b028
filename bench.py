"""Benchmark: optimal trajectories/s (100 AM iterations) and the CEM plan-cycle latency.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--scenes S | --scenes-per-gpu S]

Workload (BASELINE.json config 5: 4096 synthetic highway scenes, each a config-2 planning cycle):
every step is one full CEM planning cycle -- B=1000 set-point samples, 10 obstacles, 4 CEM
iterations, top-150 constraint elites / top-100 elites, 100 AM iterations, m=100 timesteps over
5 s, order-10 Bernstein basis -- for every scene.  The 4096 scenes are split over the ranks in
contiguous blocks (no collective on the data path): strong scaling, N=1 plans all 4096.
value = 4096 * 4 * 1000 trajectories / max-over-ranks device time per step.  With --gpus N and no
WORLD_SIZE in the environment the script starts its N ranks itself (torch.distributed.run).

At N > 1 it also times config 4 sharded over the ranks (one scene, B = 10 000 x 50 obstacles,
ShardedCEM with NCCL collectives and with the NVLink peer-memory exchange).  At N = 1 it adds the
config-2 cycle latency (p50/p99 through the public solve_bilevel), config 3 (CVAE warm start),
config 4 on one GPU and the closed-loop suite.

--impl reference times the reference algorithm on the host cores (the float64 numpy oracle
restatement in oracle/, one process per core): each step every core runs one CEM iteration
of the same workload on a bounded sample of B=100 samples of its own scene.
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import argparse  # noqa: E402
import json  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "optimal trajectories/sec (100 iters)"
B_CEM, N_CEM, N_CONS, N_ELITE, AM_ITERS, N_OBS, M, T = 1000, 4, 150, 100, 100, 10, 100, 5.0
F_IT = 24 * M * 11 + 15 * M * N_OBS + 60 * M + 8 * 11 * 11 + 10 * 11   # algorithmic flop / sample / AM iteration
REF_B = 100


# ----------------------------------------------------------------------------- reference arm (host)
def _ref_worker(args):
    """One CEM iteration (sample -> stage-1 -> 100-iteration AM -> rank -> refit) of the
    oracle restatement on B samples of scene `seed` (pkg/bilevel.py:249-292)."""
    seed, B = args
    import oracle as O
    from paper_2212_02224_b200.scenes import highway_scene
    sc = highway_scene(seed)
    sp = sc.spec
    _, W, Wd, Wdd = O.basis_matrices(10, M, T)
    qp = O.tracking_qp(W, Wd, Wdd, 4)
    aug = O.aug_qp(W, Wd, Wdd, qp.A_eq, N_OBS, 1.0)
    lim = O.Limits(sp.obstacles_x, sp.obstacles_y, sp.ellipse_a, sp.ellipse_b, sp.v_max, sp.a_max, sp.kappa_max,
                   sp.c_max, sp.y_lb, sp.y_ub, sp.v_min)
    x0 = sc.initial_state
    mean = np.concatenate([np.full(4, x0[1]), np.full(4, np.hypot(x0[2], x0[3]))])
    cov = np.diag(np.concatenate([np.full(4, 1.5 ** 2), np.full(4, 3.0 ** 2)]))
    t0 = time.perf_counter()
    O.cem_cycle(qp, aug, W, Wd, Wdd, x0, lim, mean, cov, batch=B, n_cons=min(N_CONS, B), n_elite=min(N_ELITE, B),
                iters=1, eta=0.7, gamma=0.9, w_res=1.0, rng=np.random.default_rng(seed), am_iters=AM_ITERS)
    return time.perf_counter() - t0


# Per-core speed of the port against the reference itself, measured once on one host
# (tools/ref_vs_port.py -> profiles/r02/ref_vs_port.json): the port is the faster of the two, so
# the reported CPU baseline is conservative.
REF_VS_PORT = os.path.join(ROOT, "profiles", "r02", "ref_vs_port.json")


def cpu_reference(steps: int, warmup: int, cores: int | None = None, batch: int = REF_B):
    import multiprocessing as mp
    cores = cores or os.cpu_count() or 1
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(cores) as pool:
        for s in range(warmup + steps):
            t0 = time.perf_counter()
            pool.map(_ref_worker, [(1000 * s + c, batch) for c in range(cores)])
            if s >= warmup:
                times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    out = {"value": cores * batch / t, "unit": "trajectories/s", "cores": cores, "kind": "port",
           "sample": f"per step: {cores} processes x one CEM iteration (B={batch}, 10 obstacles, 100 AM iterations, "
                     f"rank+refit) of the float64 oracle restatement; {steps} steps after {warmup} warm-up, "
                     f"{t:.2f} s/step"}
    if os.path.exists(REF_VS_PORT):
        with open(REF_VS_PORT) as fh:
            rv = json.load(fh)
        out["port_vs_reference_per_core"] = rv.get("port_over_reference")
    return out, t


def run_reference(args, rank: int, world: int, dist):
    ranks = world
    if dist is not None:                   # every rank checks in (the launcher test counts them)
        import torch
        seen = torch.ones(1)
        dist.all_reduce(seen)
        ranks = int(seen.item())
    if rank != 0:
        return
    ref, t = cpu_reference(args.steps, args.warmup, args.ref_cores, args.ref_batch)
    line = {"metric": METRIC, "value": ref["value"], "unit": ref["unit"], "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"CEM iteration on host cores, B={args.ref_batch} samples per core, 10 obstacles, "
                                   "100 AM iterations, m=100, order-10 Bernstein"},
            "impl": "reference", "cpu_baseline": ref, "ranks": ranks,
            "e2e": {"value": ref["value"], "unit": ref["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- B200 arm
class ClockSampler:
    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except (ValueError, IndexError):
                continue
            for nm, flag in zip(names, parts[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_planner(device: int):
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.fleet import FleetPlanner
    basis = bd.build_basis(10, M, T, "bernstein")
    cfg = bd.BiLevelConfig(B_CEM, N_CONS, N_ELITE, N_CEM, 0.7, 0.9, 1.0)
    return FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, AM_ITERS, 1e-3),
                        N_OBS, cfg, device=device)


def cem_latency(device: int, cycles: int = 120):
    """Single-scene config-2 cycle through the public drop-in solve_bilevel (host numpy in/out)."""
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.scenes import highway_scene
    basis = bd.build_basis(10, M, T, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4),
                                 bd.ProjectionConfig(1.0, AM_ITERS, 1e-3), N_OBS, device=device)
    scene = highway_scene(0)
    mean, cov = initial_distribution(scene)
    cfg = bd.BiLevelConfig(B_CEM, N_CONS, N_ELITE, N_CEM, 0.7, 0.9, 1.0, mean, cov)
    for s in range(3):
        bd.solve_bilevel(scene, solver, cfg, np.random.default_rng(s))
    ts = []
    for s in range(cycles):
        rng = np.random.default_rng(100 + s)
        t0 = time.perf_counter()
        res = bd.solve_bilevel(scene, solver, cfg, rng)
        ts.append(1e3 * (time.perf_counter() - t0))
        assert np.isfinite(res.best.upper_cost)
    # the same cycle with the draws on the device (FleetPlanner.plan, device Philox): no host RNG
    from paper_2212_02224_b200.fleet import FleetPlanner
    fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, AM_ITERS, 1e-3), N_OBS,
                      bd.BiLevelConfig(B_CEM, N_CONS, N_ELITE, N_CEM, 0.7, 0.9, 1.0), device=device)
    for s in range(3):
        fp.plan([scene], seed=s)
    td = []
    for s in range(cycles):
        t0 = time.perf_counter()
        r = fp.plan([scene], seed=100 + s)
        td.append(1e3 * (time.perf_counter() - t0))
        assert np.isfinite(r.best_cost[0])
    return {"p50_ms": float(np.percentile(ts, 50)), "p99_ms": float(np.percentile(ts, 99)), "cycles": cycles,
            "config": "B=1000, 10 obstacles, 4 CEM iterations, n=150, q=100, 100 AM iterations; host call to "
                      "host-visible best xi via solve_bilevel (numpy Generator draws, H2D+D2H included)",
            "device_rng": {"p50_ms": float(np.percentile(td, 50)), "p99_ms": float(np.percentile(td, 99)),
                           "api": "FleetPlanner.plan (device Philox draws), host call to host-visible results"}}


def cvae_config3(device: int, cycles: int = 120):
    """BASELINE config 3: CVAE decoder draws 1000 set-points from a scene embedding (the 55-entry
    observation), which warm-start iteration 1 of the config-2 CEM cycle; p50 of decode + cycle
    through the public API (tcgen05 decoder, synthetic seeded weights: the reference ships none)."""
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.cvae import CVAEDecoder
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.scenes import highway_scene, spawn_worlds
    from paper_2212_02224_b200.worlds import PlannerEnv, build_scenes
    basis = bd.build_basis(10, M, T, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4),
                                 bd.ProjectionConfig(1.0, AM_ITERS, 1e-3), N_OBS, device=device)
    scene = highway_scene(0)
    mean, cov = initial_distribution(scene)
    cfg = bd.BiLevelConfig(B_CEM, N_CONS, N_ELITE, N_CEM, 0.7, 0.9, 1.0, mean, cov)
    dec = CVAEDecoder.synthetic(0, context=solver.context)
    # the scene embedding: observe() of the world, built on the device
    *_, obs = build_scenes(solver.context, basis, spawn_worlds([0]), PlannerEnv(), outputs=True)
    solver.projector._scene_key = None
    raw = dec.decode(obs[0], np.random.default_rng(0).standard_normal((B_CEM, 2)))
    shift = mean - raw.mean(axis=0)            # untrained decoder: centre its output on the prior mean
    ts = []
    for s in range(cycles + 3):
        rng = np.random.default_rng(200 + s)
        t0 = time.perf_counter()
        ws = dec.warm_start(obs[0], B_CEM, solver.layout, rng, shift=shift)
        res = bd.solve_bilevel(scene, solver, cfg, rng, warm_start=ws)
        if s >= 3:
            ts.append(1e3 * (time.perf_counter() - t0))
        assert not res.degraded
    return {"p50_ms": float(np.percentile(ts, 50)), "p99_ms": float(np.percentile(ts, 99)), "cycles": cycles,
            "config": "CVAE decode of 1000 set-points (tcgen05 bf16 hidden layers) + config-2 CEM cycle warm-started "
                      "from them (rows stay on the device: bd_cvae_warm_start); host call to host-visible best xi"}


def dense_config4(device: int, steps: int = 3):
    """BASELINE config 4 on one GPU: one scene, B = 10 000 samples x 50 obstacles, one full CEM
    cycle (4 iterations, 100 AM iterations) per step, device Philox draws."""
    import torch
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.fleet import FleetPlanner, initial_distribution
    from paper_2212_02224_b200.scenes import HighwayRecipe, highway_scene
    basis = bd.build_basis(10, M, T, "bernstein")
    cfg = bd.BiLevelConfig(10_000, N_CONS, N_ELITE, N_CEM, 0.7, 0.9, 1.0)
    fp = FleetPlanner(basis, bd.TrackingWeights(), bd.ParamLayout(4), bd.ProjectionConfig(1.0, AM_ITERS, 1e-3), 50,
                      cfg, device=device)
    sc = highway_scene(0, HighwayRecipe(density=3.0, vehicle_count=80, n_obs=50, obstacle_range=250.0))
    fp.set_scenes([sc])
    mean, cov = initial_distribution(sc)
    m_t = torch.tensor(mean[None], dtype=torch.float64, device=device)
    c_t = torch.tensor(cov[None], dtype=torch.float64, device=device)
    stream = torch.cuda.current_stream(device)
    fp.context.set_stream(stream.cuda_stream)
    outs = {"best_cost": torch.zeros(1, dtype=torch.float64, device=device),
            "iterations_done": torch.zeros(1, dtype=torch.int32, device=device)}
    fp.plan_device(1, 0, m_t, c_t, outs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(steps):
        fp.plan_device(1, 1 + k, m_t, c_t, outs)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    assert int(outs["iterations_done"][0]) == N_CEM
    return {"value": 10_000 * N_CEM / (ms / 1e3), "unit": "trajectories/s", "cycle_ms": ms,
            "config": "1 scene, B=10000, 50 obstacles, 4 CEM iterations, 100 AM iterations (1 GPU)"}


def closed_loop_suite(device: int, episodes: int = 256, length: int = 150):
    """a fleet of closed-loop episodes (run_episode semantics, replan every 5 ticks)
    with the reference planner's default configuration (PlannerEnvConfig: B=250, N=5, m=50 over 10 s,
    6 obstacles, 50 AM iterations): device scene build -> CEM -> controls -> simulator, one batched
    call per replan instant.  Host wall clock around the whole run (logs included)."""
    from paper_2212_02224_b200.episodes import run_episodes
    from paper_2212_02224_b200.planners import PlannerEnvConfig, make_batch_planner
    from paper_2212_02224_b200.sim import RoadSpec, ScenarioConfig
    scs = [ScenarioConfig(RoadSpec(4), 1.0, 12, s, episode_length=length) for s in range(episodes)]
    planner = make_batch_planner("mpc-bilevel", PlannerEnvConfig(), device=device)
    run_episodes(scs[:4], planner, device=f"cuda:{device}")            # warm-up (allocations, first launches)
    walls = []
    for _ in range(3):                                                  # host wall clock: median of 3 runs
        t0 = time.perf_counter()
        logs = run_episodes(scs, planner, device=f"cuda:{device}")
        walls.append(time.perf_counter() - t0)
    wall = float(np.median(walls))
    ticks = sum(len(lg.steps) for lg in logs)
    cycles = sum(len(lg.plan_records) for lg in logs)
    return {"episodes_per_s": episodes / wall, "ticks_per_s": ticks / wall, "plans_per_s": cycles / wall,
            "wall_s": wall, "ticks": ticks, "collisions": sum(lg.collided for lg in logs),
            "failures": sum(lg.failed for lg in logs),
            "config": f"{episodes} episodes x {length} ticks (dt 0.1 s, replan every 5), 4-lane highway, density 1, 12 "
                      "neighbours; mpc-bilevel with PlannerEnvConfig defaults; host wall clock incl. step records, median of 3 runs"}


def sharded_config4(dev: int, rank: int, world: int, dist, steps: int = 2):
    """BASELINE config 4 sharded over the ranks: one scene, B = 10 000 samples x 50 obstacles, 4 CEM
    iterations x 100 AM iterations per cycle (ShardedCEM, parallel.py).  Two exchange modes: NCCL
    collectives (all-reduce of the iteration maxima, all-gather of residual/cost, best-row sum) and
    the NVLink peer-memory exchange fused into the AM epilogue (P2PExchange).  Device time of a
    whole cycle, max over ranks."""
    import torch
    import paper_2212_02224_b200 as bd
    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.parallel import CudaShardBackend, P2PExchange, ShardedCEM
    from paper_2212_02224_b200.scenes import HighwayRecipe, highway_scene
    B = 10_000
    basis = bd.build_basis(10, M, T, "bernstein")
    solver = bd.LowerLevelSolver(basis, bd.TrackingWeights(), bd.ParamLayout(4),
                                 bd.ProjectionConfig(1.0, AM_ITERS, 1e-3), 50, device=dev)
    sc = highway_scene(0, HighwayRecipe(density=3.0, vehicle_count=80, n_obs=50, obstacle_range=250.0))
    mean, cov = initial_distribution(sc)
    be = CudaShardBackend(solver, sc, device=dev)
    stream = torch.cuda.current_stream(dev)
    out = {"config": f"1 scene, B={B}, 50 obstacles, {N_CEM} CEM iterations x {AM_ITERS} AM iterations, batch "
                     f"sharded over {world} GPU(s) ({B // world} samples each)"}
    best = {}
    for mode in ("nccl", "p2p"):
        try:
            ex = P2PExchange(solver.context, B, AM_ITERS) if mode == "p2p" else None
            kw = dict(batch=B, n_cons=N_CONS, n_elite=N_ELITE, iterations=N_CEM, eta=0.7, gamma=0.9,
                      residual_weight=1.0, am_iters=AM_ITERS, tol=1e-3, exchange=ex)
            ShardedCEM(be, seed=1, **kw).run(mean, cov)                      # warm-up
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for k in range(steps):
                res = ShardedCEM(be, seed=2 + k, **kw).run(mean, cov)
            e1.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            best[mode] = (res.best_index, res.best_xi.tobytes())
            out[mode] = {"value": B * N_CEM / (ms / 1e3), "unit": "trajectories/s", "cycle_ms": ms,
                         "best_index": res.best_index}
        except Exception as exc:  # noqa: BLE001  (reported in the line, the fleet number stands)
            out[mode] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if len(best) == 2:
        out["modes_agree"] = best["nccl"] == best["p2p"]
    return out


def comm_info():
    """NCCL communicator facts for the line (NCCL_DEBUG=INFO prints the init log on stderr)."""
    import torch
    try:
        v = torch.cuda.nccl.version()
        return {"nccl_version": ".".join(map(str, v)) if isinstance(v, tuple) else str(v),
                "nccl_debug": os.environ.get("NCCL_DEBUG")}
    except Exception as exc:  # noqa: BLE001
        return {"error": str(exc)[:200]}


def run_b200(args, rank: int, world: int, dist):
    import torch

    from paper_2212_02224_b200.fleet import initial_distribution
    from paper_2212_02224_b200.parallel import shard_range
    from paper_2212_02224_b200.scenes import highway_scene

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    if args.scenes_per_gpu:                            # weak scaling: fixed scenes per GPU
        total, scaling = args.scenes_per_gpu * world, "weak"
    else:                                              # strong scaling: the whole config-5 job split
        total, scaling = args.scenes, "strong"
    lo, hi, _ = shard_range(total, rank, world)
    S = hi - lo
    planner = make_planner(dev)
    ctx = planner.context
    stream = torch.cuda.Stream(device=dev)       # a real (non-null) stream shared by the library and the events
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    scenes = [highway_scene(lo + j) for j in range(S)]
    planner.set_scenes(scenes)
    mc = [initial_distribution(sc) for sc in scenes]
    mean = torch.tensor(np.stack([m for m, _ in mc]), dtype=torch.float64, device=dev)
    cov = torch.tensor(np.stack([c for _, c in mc]), dtype=torch.float64, device=dev)
    outs = {"best_index": torch.zeros(S, dtype=torch.int64, device=dev),
            "best_xi": torch.zeros(S, 22, dtype=torch.float64, device=dev),
            "best_cost": torch.zeros(S, dtype=torch.float64, device=dev),
            "iterations_done": torch.zeros(S, dtype=torch.int32, device=dev)}
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    peaks = {"fp32_tflops": ctx.probe("fp32_tflops"), "fp32x2_tflops": ctx.probe("fp32x2_tflops")}
    fp32_peak = max(peaks.values())

    for w in range(args.warmup):
        planner.plan_device(S, 7 + w, mean, cov, outs, scene_offset=lo)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ctx.set_option("timing", 1)
    ctx.stat("reset")
    launches0 = ctx.launches()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.zero_()                       # L2 flush between timed steps (outside the events)
            ev[k][0].record(stream)
            planner.plan_device(S, 1000 + k, mean, cov, outs, scene_offset=lo)
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ctx.set_option("timing", 0)
    launches = ctx.launches() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(np.sum(step_ms))
    am_ms = ctx.stat("am_ms")
    am_n = ctx.stat("am_launches")
    am_si = ctx.stat("am_sample_iters")
    done = outs["iterations_done"].cpu().numpy()
    assert np.all(done == N_CEM), f"CEM cycles incomplete: {done}"
    assert torch.isfinite(outs["best_cost"]).all()
    t_max = total_ms
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    traj = total * N_CEM * B_CEM * args.steps
    value = traj / (t_max / 1e3)

    # end to end through the public API: the planning cycle of MPCBiLevelPlanner.plan_cycle for
    # this rank's worlds -- host world state in (H2D), device scene build, CEM cycle, control
    # emission, host controls + best records out (D2H), every step
    from paper_2212_02224_b200.scenes import spawn_worlds
    from paper_2212_02224_b200.worlds import ControlEmitter, PlannerEnv
    worlds = spawn_worlds(range(10_000 + lo, 10_000 + hi))
    emitter = ControlEmitter(ctx, planner.solver.basis, T, 0.1, PlannerEnv())
    ctx.set_stream(None)
    planner.plan_cycle(worlds, PlannerEnv(), emitter, seed=1)      # warm the host path
    torch.cuda.synchronize()
    e2e_steps = max(1, min(args.steps, 5))
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        acc, ste, sing, res = planner.plan_cycle(worlds, PlannerEnv(), emitter, seed=2 + k,
                                                 scene_offset=10_000 + lo)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    assert np.all(res.iterations_done == N_CEM)
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = worlds.ego.nbytes + worlds.veh.nbytes + worlds.n_veh.nbytes + worlds.road.nbytes + M * 8 + S * (8 + 64) * 8
    d2h = res.best_index.nbytes + res.best_params.nbytes + res.best_xi.nbytes + 3 * S * 8 + res.stats.nbytes + \
        res.final_mean.nbytes + res.final_cov.nbytes + res.iterations_done.nbytes + acc.nbytes + ste.nbytes + S * 4 + S * 6 * 8

    sharded = sharded_config4(dev, rank, world, dist) if world > 1 else None
    if rank != 0:
        return
    am_avg_ms = am_ms / max(am_n, 1.0)
    flop_per_launch = F_IT * am_si / max(am_n, 1.0)
    achieved = flop_per_launch / (am_avg_ms * 1e-3) / 1e12
    prof = {}
    tpath = os.path.join(ROOT, "profiles", "am_kernel_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            prof = json.load(fh)
    executed = prof.get("executed_fp32_flop_per_sample_iter")
    line = {
        "metric": METRIC, "value": value, "unit": "trajectories/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic highway scenes (seeded spawn_world+build_scene recipe), device Philox set-point draws",
        "config": {"workload": f"CEM plan cycles: {total} scenes over {world} GPU(s) x (B=1000 samples, 10 obstacles, "
                               "4 CEM iterations, top-150/top-100 elites, 100 AM iterations, m=100 over 5 s, "
                               "order-10 Bernstein)",
                   "scenes": total, "scenes_per_gpu": S, "batch": B_CEM, "cem_iterations": N_CEM,
                   "am_iterations": AM_ITERS, "obstacles": N_OBS,
                   "parallelism": f"scenes sharded over {world} GPU(s) in contiguous blocks, no data-path collective",
                   "l2": "flushed (256 MB write) between timed steps"},
        "e2e": {"value": total * N_CEM * B_CEM / e2e_s, "unit": "trajectories/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "api": "FleetPlanner.plan_cycle (host world state -> device scene build -> CEM cycle -> control "
                       "emission -> host controls + best records)"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp32_peak, "traffic": prof.get("dram_bytes_per_launch"),
                     "kernel": "am_kernel (fused AM projection)", "flop_per_launch": flop_per_launch,
                     "avg_launch_ms": am_avg_ms, "kernel_share_of_step": am_ms / max(total_ms, 1e-9),
                     "peak_probes": peaks,
                     "peak_source": "max of the live FFMA and FFMA2 (fma.rn.f32x2) issue probes (bd_probe); "
                                    "MEASURED_PEAKS.json has no FP32 CUDA-core figure",
                     "executed_fp32_flop_per_sample_iter": executed,
                     "executed_frac": (achieved * executed / F_IT / fp32_peak) if executed else None,
                     "executed_source": prof.get("executed_source")},
        "clocks": clk.summary(),
    }
    if world > 1:
        line["sharded_config4"] = sharded
        line["comm"] = comm_info()
    if world == 1:
        line["cem_cycle_latency"] = cem_latency(dev)
        line["dense_config4"] = dense_config4(dev)
        line["cvae_config3_latency"] = cvae_config3(dev)
        line["closed_loop_suite"] = closed_loop_suite(dev)
        ref, _ = cpu_reference(args.steps, args.warmup, args.ref_cores, args.ref_batch)
        line["cpu_baseline"] = ref
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scenes", type=int, default=4096)            # BASELINE config 5: 4096 scenes per job
    ap.add_argument("--scenes-per-gpu", type=int, default=None)    # weak-scaling alternative
    ap.add_argument("--ref-batch", type=int, default=REF_B)        # reference arm: samples per core per step
    ap.add_argument("--ref-cores", type=int, default=None)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: start the ranks ourselves (same command under torch.distributed.run)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        if args.impl == "b200":
            os.environ.setdefault("NCCL_DEBUG", "INFO")            # communicator init log (stderr)
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            local = int(os.environ.get("LOCAL_RANK", 0))
            torch.cuda.set_device(local)
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group("gloo")
        dist = tdist
    if args.impl == "reference":
        run_reference(args, rank, world, dist)
    else:
        from paper_2212_02224_b200.build import LIB, build
        if rank == 0 and not os.path.exists(LIB):
            build()
        if dist is not None:
            dist.barrier()
        run_b200(args, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
