"""Benchmark: batched fp64 Helmholtz + biharmonic solves (BASELINE config 4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c4|c5:N|c1|c3|step] [--kx-rows R]

One step = HelmholtzLU.solve + BiharmonicLU.solve over this rank's kx slab of
the 2048 x 1025 wavenumber plane (n_x = 1024, nu = 1/2000, dt = 1e-4),
complex128 N(0,1) right-hand sides resident in HBM (34 GB each at N = 1, far
larger than L2, so no flush is needed between steps).  The LU objects are
built once before timing, as the reference's stepper does (build time is
reported separately).  Multi-GPU: one process per GPU, kx slabs, no
collectives on the data path (weak scaling of the wavenumber plane would be
'strong' here: the plane is fixed and split -- see "scaling").

--config c3 is BASELINE config 3 (transforms + solves on a 257 x 256 x 256
field); with --gpus N > 1 it runs on x-plane / kx-row slabs with the exchange
fused into the plane FFT kernels over peer memory (run_c3_slab).

The reference arm (--impl reference) times the oracle port of the reference
CPU algorithm (numpy, identical arithmetic) on all host cores over kx slabs.
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

NU_C4, DT_C4 = 1 / 2000, 1e-4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--kx-rows", type=int, default=0, help="limit the kx rows per rank (debug)")
    ap.add_argument("--kx-fold", type=int, default=0,
                    help="profile subset: the rows of rank 0 of a K-way folded split (keeps mirror pairs)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU check of the multi-rank launch: gloo ranks, folded slabs, max-over-ranks "
                         "timing, oracle solves instead of the device (no GPU needed; not a bench number)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--method", default="stream", choices=["stream", "stored"])
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the timed step from a CUDA graph (auto: launch-bound sizes only)")
    return ap.parse_args()


def workload(cfg: str):
    """(name, n_x, n_y, n_z, nu, dt)"""
    if cfg == "c4":
        return "config4: n_x=1024 (N=1025), 2048x1025 wavenumbers, nu=1/2000, dt=1e-4", 1024, 2048, 2048, NU_C4, DT_C4
    if cfg.startswith("c5:"):
        N = int(cfg[3:])
        return f"config5: N={N}, 512x257 wavenumbers, nu=1/2000, dt=1e-4", N - 1, 512, 512, NU_C4, DT_C4
    if cfg == "c1":
        return "config1/2: n_x=63, 64x33 wavenumbers, nu=dt=1e-3", 63, 64, 64, 1e-3, 1e-3
    raise SystemExit(f"unknown config {cfg}")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def measured_traffic(cfg, method, op, unknowns):
    """DRAM bytes (read + write) per launch of the dominant kernel, from the
    committed ncu --set full capture (profiles/traffic_c4.json: bytes per
    unknown of the full config-4 launches, scaled to this launch's unknowns)."""
    path = os.path.join(ROOT, "profiles", "traffic_c4.json")
    if cfg != "c4" or method != "stream" or not os.path.exists(path):
        return None, None
    try:
        t = json.load(open(path))[op]
        return float(t["bytes_per_unknown"]) * unknowns, f"{t['source']} ({t['bytes_per_unknown']:.1f} B/unknown)"
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        if os.environ.get("SHEN_BENCH_NO_CLOCKS"):  # diagnosis only: the bench line then says "unsampled"
            self.proc = None
            return self
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        # start timing only once nvidia-smi has initialised NVML and written a
        # sample: its start-up takes driver locks that can stall CUDA launches
        # (a host-bound timed region of a few ms would absorb the whole stall)
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < 10.0:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                pass
            time.sleep(0.05)
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows]
        smax = float(rows[0][2])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        loaded = [s for s in sm if s > 0.5 * smax] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


# ======================================================================= B200 arm

def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_1701_03787_b200 import solvers as S
    from paper_1701_03787_b200.matrices import assemble
    from paper_1701_03787_b200.mesh import channel_z2

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name, n_x, n_y, n_z, nu, dt = workload(args.config)
    z2_full = channel_z2(n_y, n_z)
    from paper_1701_03787_b200.shard import kx_rows_folded, kx_slab

    if args.kx_rows:  # debug slab: contiguous rows
        lo, hi = kx_slab(n_y, rank, world)
        rows = np.arange(lo, min(hi, lo + args.kx_rows))
    elif args.kx_fold:  # profiling subset with mirror pairs
        rows = kx_rows_folded(n_y, 0, args.kx_fold)
    else:  # folded slabs: whole (m, -m) pairs per rank (the biharmonic solves them together)
        rows = kx_rows_folded(n_y, rank, world)
    lo, hi = 0, len(rows)
    z2 = np.ascontiguousarray(z2_full[rows])
    mats = assemble(n_x, 0)
    dev = torch.device("cuda", local)

    t0 = time.perf_counter()
    hlu = S.build_helmholtz(mats, nu, dt, z2, method=args.method)
    blu = S.build_biharmonic(mats, nu, dt, z2, method=args.method)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    # device-timed build (second build, warm)
    eb0, eb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eb0.record()
    hlu = S.build_helmholtz(mats, nu, dt, z2, method=args.method)
    blu = S.build_biharmonic(mats, nu, dt, z2, method=args.method)
    eb1.record()
    torch.cuda.synchronize()
    build_ms = eb0.elapsed_time(eb1)

    B = z2.size
    nh, nb = mats.n_dir, mats.n_bih
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    fh = torch.randn((nh, B), dtype=torch.complex128, device=dev, generator=gen).mul_(np.sqrt(2.0))
    fb = torch.randn((nb, B), dtype=torch.complex128, device=dev, generator=gen).mul_(np.sqrt(2.0))
    xh = torch.empty_like(fh)
    xb = torch.empty_like(fb)

    def step(evs=None):
        if evs is not None:
            evs[0].record()
        hlu.solve_into(fh, xh, True)
        if evs is not None:
            evs[1].record()
        blu.solve_into(fb, xb, True)
        if evs is not None:
            evs[2].record()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    # launch-bound sizes (config 1/2: tens of microseconds per solve): the
    # step is captured once into a CUDA graph and replayed, so the host-side
    # launch path is out of the timed loop
    use_graph = args.graph == "on" or (args.graph == "auto" and B * (nh + nb) < 50_000_000)
    graph = None
    if use_graph:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step()
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record()
        for k in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                step(evs[k])
        t_end.record()
        torch.cuda.synchronize()
    total_ms = t_start.elapsed_time(t_end)
    if graph is not None:  # per-operator times from a separate eager pass
        for k in range(args.steps):
            step(evs[k])
        torch.cuda.synchronize()
    h_all = [e[0].elapsed_time(e[1]) for e in evs]
    b_all = [e[1].elapsed_time(e[2]) for e in evs]
    h_ms, b_ms = float(np.mean(h_all)), float(np.mean(b_all))
    if world > 1:
        t = torch.tensor([total_ms, h_ms, b_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, h_ms, b_ms = t.tolist()
        bt = torch.tensor([B], dtype=torch.int64, device=dev)
        dist.all_reduce(bt)
        B_all = int(bt.item())
    else:
        B_all = B
    unk_h = nh * B_all
    unk_b = nb * B_all
    value = (unk_h + unk_b) * args.steps / (total_ms / 1e3)

    # correctness spot check on this rank (sampled systems vs the oracle)
    parity = spot_parity(mats, nu, dt, z2, fh, xh, fb, xb) if rank == 0 else None

    peak, peak_src = measured_peak()
    traffic, traffic_src = measured_traffic(args.config, args.method, "biharmonic" if b_ms >= h_ms else "helmholtz",
                                            (nb if b_ms >= h_ms else nh) * B)
    bytes_h = 32.0 * nh * B  # per launch on this rank
    bytes_b = 32.0 * nb * B
    ach_h = bytes_h / (h_ms / 1e3) / 1e9
    ach_b = bytes_b / (b_ms / 1e3) / 1e9
    dom = "biharmonic" if b_ms >= h_ms else "helmholtz"
    ach = ach_b if dom == "biharmonic" else ach_h
    ckpt_bytes_h = 8.0 * hlu._ckpt.numel() if hlu._ckpt is not None else 0.0
    ckpt_bytes_b = 8.0 * blu._ckpt.numel() if blu._ckpt is not None else 0.0
    # the timed arrays (137 GB at config 4) are done with: free them before the
    # end-to-end sample allocates its own LU objects and pipeline buffers
    del fh, fb, xh, xb, hlu, blu
    torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:
        # every rank streams its own sample through the public API (its own
        # PCIe link); the value is the sum of the ranks' unknowns over the
        # slowest rank's time
        e2e = run_e2e(S, mats, nu, dt, z2_full[rows], args, world)
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        cpu = cpu_baseline(mats, nu, dt, z2_full)
    if rank == 0:
        line = {
            "metric": "solved unknowns/s (batched fp64 Helmholtz+biharmonic); % of HBM roofline",
            "value": value,
            "unit": "unknowns/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(args.warmup, 3),
            "ms_per_step": total_ms / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64 (complex128 RHS/solution)",
            "data": "synthetic: complex128 N(0,1) RHS (torch Philox, seed 1234+rank), z2 of the channel plane",
            "config": {"workload": name, "systems_total": int(B_all), "kx_rows_per_rank": int(hi - lo),
                       "modes": {"helmholtz": nh, "biharmonic": nb}, "parallelism": f"kx-slab x{world} (folded: (m, -m) pairs per rank)",
                       "l2_policy": "inputs (34 GB/operator at N=1) >> 126 MB L2; no flush needed",
                       "lu": "built once before timing (stepper usage); build timed separately",
                       "method": args.method, "cuda_graph": bool(graph is not None)},
            "per_operator": {
                "helmholtz": {"ms": h_ms, "ms_median": float(np.median(h_all)), "ms_best": float(np.min(h_all)),
                              "unknowns_per_s": nh * B / (h_ms / 1e3), "GBps_alg": ach_h,
                              "frac": ach_h / peak, "ckpt_read_bytes": ckpt_bytes_h},
                "biharmonic": {"ms": b_ms, "ms_median": float(np.median(b_all)), "ms_best": float(np.min(b_all)),
                               "unknowns_per_s": nb * B / (b_ms / 1e3), "GBps_alg": ach_b,
                               "frac": ach_b / peak, "ckpt_read_bytes": ckpt_bytes_b},
            },
            "roofline": {"bound": "hbm", "kernel": f"{dom} {args.method} solve", "achieved": ach, "peak": peak,
                         "unit": "GB/s", "frac": ach / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         "algorithmic_bytes": "32 B per complex unknown (16 B RHS read + 16 B solution write)"},
            "build_ms": build_ms,
            "build_wall_s_first": build_s,
            "parity": parity,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": 2 * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def spot_parity(mats, nu, dt, z2, fh, xh, fb, xb):
    from oracle import shen_oracle as O

    flat = z2.reshape(-1)
    idx = np.unique(np.concatenate([np.argsort(flat)[-4:], np.linspace(0, flat.size - 1, 12).astype(int)]))
    z = flat[idx]
    it = __import__("torch").from_numpy(idx).to(fh.device)
    f1 = fh[:, it].cpu().numpy()
    x1 = xh[:, it].cpu().numpy()
    f2 = fb[:, it].cpu().numpy()
    x2 = xb[:, it].cpu().numpy()
    rh = O.helmholtz_solve(O.helmholtz_factor(mats, nu, dt, z), f1)
    rb = O.biharmonic_solve(O.biharmonic_factor(mats, nu, dt, z), f2)
    resid = max(float(O.residual_longdouble(O.dense_biharmonic(mats, nu, dt, z[j]), x2[:, j], f2[:, j]))
                for j in range(len(z)))
    resid_ref = max(float(O.residual_longdouble(O.dense_biharmonic(mats, nu, dt, z[j]), rb[:, j], f2[:, j]))
                    for j in range(len(z)))
    return {"systems_checked": int(len(z)), "helmholtz_max_rel": float(O.max_rel_per_system(x1, rh).max()),
            "biharmonic_max_rel": float(O.max_rel_per_system(x2, rb).max()),
            "biharmonic_residual_max": resid, "reference_residual_max_same_systems": resid_ref}


def run_e2e(S, mats, nu, dt, z2_rank, args, world=1):
    """Same metric through the public API with HOST buffers: page-locked numpy
    arrays in and out (the application's own buffers), so every step copies
    the RHS host->device and the solution device->host; the API pipelines the
    copies against the solve in column slabs.  Bounded sample per rank: the
    first 256 of the rank's kx rows (262,400 systems; 4.3 GB per operator
    RHS).  With N ranks each rank runs its own sample concurrently (one PCIe
    link per GPU); timing is max over ranks after a barrier, unknowns summed."""
    import torch
    import torch.distributed as dist

    rows = min(256, z2_rank.shape[0])
    z2 = np.ascontiguousarray(z2_rank[:rows])
    hlu = S.build_helmholtz(mats, nu, dt, z2, method=args.method)
    blu = S.build_biharmonic(mats, nu, dt, z2, method=args.method)

    def pinned(shape):
        return torch.empty(shape, dtype=torch.complex128, pin_memory=True).numpy()

    shp_h, shp_b = (mats.n_dir,) + z2.shape, (mats.n_bih,) + z2.shape
    fh, fb, xh, xb = pinned(shp_h), pinned(shp_b), pinned(shp_h), pinned(shp_b)
    g = torch.Generator().manual_seed(5)
    fh[...] = torch.randn(shp_h, dtype=torch.complex128, generator=g).numpy()
    fb[...] = torch.randn(shp_b, dtype=torch.complex128, generator=g).numpy()
    jobs = [(hlu, fh, xh), (blu, fb, xb)]
    for _ in range(2):
        S.solve_many(jobs)
    steps = 3
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        S.solve_many(jobs)  # both operators through one host<->device pipeline
    dt_s = (time.perf_counter() - t0) / steps
    unk = (mats.n_dir + mats.n_bih) * z2.size
    h2d, d2h = int(fh.nbytes + fb.nbytes), int(xh.nbytes + xb.nbytes)
    if world > 1:
        t = torch.tensor([dt_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        c = torch.tensor([unk, h2d, d2h], dtype=torch.int64, device="cuda")
        dist.all_reduce(c)
        dt_s = float(t.item())
        unk, h2d, d2h = (int(v) for v in c.tolist())
    return {"value": unk / dt_s, "unit": "unknowns/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "sample": f"{world} rank(s) x {rows} kx rows x {z2.shape[1]} systems, page-locked numpy in/out",
            "ranks": world,
            "path": "solvers.solve_many([(hlu, fh, xh), (blu, fb, xb)]) (host wall clock incl. copies, "
                    "max over ranks)"}


def cpu_baseline(mats, nu, dt, z2_full):
    """Oracle port (numpy, reference arithmetic) on one host core, bounded
    sample of the same workload: 48 kx rows x 1025 systems."""
    from oracle import shen_oracle as O

    rows = 48
    z2 = np.ascontiguousarray(z2_full[:rows])
    rng = np.random.default_rng(6)
    fh = rng.standard_normal((mats.n_dir,) + z2.shape) + 1j * rng.standard_normal((mats.n_dir,) + z2.shape)
    fb = rng.standard_normal((mats.n_bih,) + z2.shape) + 1j * rng.standard_normal((mats.n_bih,) + z2.shape)
    fh_f = O.helmholtz_factor(mats, nu, dt, z2)
    fb_f = O.biharmonic_factor(mats, nu, dt, z2)
    t0 = time.perf_counter()
    O.helmholtz_solve(fh_f, fh)
    O.biharmonic_solve(fb_f, fb)
    t = time.perf_counter() - t0
    unk = (mats.n_dir + mats.n_bih) * z2.size
    return {"value": unk / t, "unit": "unknowns/s", "cores": 1, "kind": "port",
            "sample": f"{z2.shape[0]} kx rows x {z2.shape[1]} systems of the same plane, solve only (LU prebuilt), "
                      "1 thread"}


def run_dry(args):
    """The launcher and reduction logic of run_b200 on CPU: gloo process
    group, each rank's folded kx rows, the oracle's solves as the per-rank
    work, barrier + max-over-ranks time, summed systems; prints the same kind
    of JSON line (marked dry_run).  Used by tests/test_bench_launch.py."""
    import torch
    import torch.distributed as dist

    from oracle import shen_oracle as O
    from paper_1701_03787_b200.matrices import assemble
    from paper_1701_03787_b200.mesh import channel_z2
    from paper_1701_03787_b200.shard import kx_rows_folded

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    name, n_x, n_y, n_z, nu, dt = workload(args.config)
    rows = kx_rows_folded(n_y, rank, world)
    z2 = np.ascontiguousarray(channel_z2(n_y, n_z)[rows])
    mats = assemble(n_x, 0)
    rng = np.random.default_rng(1234 + rank)
    fh = rng.standard_normal((mats.n_dir,) + z2.shape) + 0j
    hf = O.helmholtz_factor(mats, nu, dt, z2)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.helmholtz_solve(hf, fh)
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    b = torch.tensor([z2.size], dtype=torch.int64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(b)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "steps": args.steps,
                          "config": {"workload": name, "systems_total": int(b.item()), "kx_rows_rank0": len(rows),
                                     "parallelism": f"kx-slab x{world} (folded: (m, -m) pairs per rank)"},
                          "ms_per_step": 1e3 * float(t.item()) / args.steps}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ======================================================================= config 3

def run_c3(args):
    """BASELINE config 3: real U(-1,1) field on the 257 x 256 x 256 mesh
    (n_x = 256, Gauss points); one step = forward Dirichlet transform ->
    Helmholtz solve per wavenumber -> inverse, then forward biharmonic
    transform -> biharmonic solve -> inverse, all on device-resident data.
    One rank: this function; several ranks: run_c3_slab (slab transforms)."""
    import torch

    from paper_1701_03787_b200 import solvers as S
    from paper_1701_03787_b200 import transforms as T
    from paper_1701_03787_b200.matrices import assemble
    from paper_1701_03787_b200.mesh import Space, build_mesh, wavenumber_grid

    rank, world, local = dist_env()
    if world > 1:
        return run_c3_slab(args)
    torch.cuda.set_device(local)
    nu, dt = 1e-3, 1e-3
    mesh = build_mesh(256, 256, 256, 2 * np.pi, np.pi)
    mats = assemble(256, 0)
    z2 = wavenumber_grid(mesh, Space.DIRICHLET).z2()
    hlu = S.build_helmholtz(mats, nu, dt, z2)
    blu = S.build_biharmonic(mats, nu, dt, z2)
    g = torch.Generator(device="cuda").manual_seed(33)
    u = (torch.rand(mesh.shape, generator=g, device="cuda", dtype=torch.float64) * 2 - 1)
    B = z2.size
    xh = torch.empty((mats.n_dir, B), dtype=torch.complex128, device="cuda")
    xb = torch.empty((mats.n_bih, B), dtype=torch.complex128, device="cuda")
    out = {}

    def step(ev=None):
        rec = (lambda i: ev[i].record()) if ev else (lambda i: None)
        rec(0)
        cd = T.forward_transform(T.PhysicalField(u, mesh), Space.DIRICHLET)
        rec(1)
        hlu.solve_into(cd.data.view(mats.n_dir, B), xh, True)
        rec(2)
        out["ud"] = T.inverse_transform(T.SpectralField(xh.view(cd.data.shape), cd.grid, mesh)).data
        rec(3)
        cb = T.forward_transform(T.PhysicalField(u, mesh), Space.BIHARMONIC)
        rec(4)
        blu.solve_into(cb.data.view(mats.n_bih, B), xb, True)
        rec(5)
        out["ub"] = T.inverse_transform(T.SpectralField(xb.view(cb.data.shape), cb.grid, mesh)).data
        rec(6)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(7)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for k in range(args.steps):
            step(evs[k])
        t1.record()
        torch.cuda.synchronize()
    total_ms = t0.elapsed_time(t1)
    names = ["forward_dirichlet", "helmholtz_solve", "inverse_dirichlet", "forward_biharmonic",
             "biharmonic_solve", "inverse_biharmonic"]
    stages = {nm: float(np.mean([e[i].elapsed_time(e[i + 1]) for e in evs])) for i, nm in enumerate(names)}
    unk = (mats.n_dir + mats.n_bih) * B
    wall = c3_wall_stages(mesh, u, B)
    cpu = None if args.no_cpu else cpu_c3()
    print(json.dumps({
        "metric": "config-3 steps/s (fwd transform + solve + inverse, Dirichlet/Helmholtz and biharmonic)",
        "value": args.steps / (total_ms / 1e3), "unit": "steps/s", "n_gpus": 1, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "none", "vs_baseline": None, "dtype": "f64 (real field, complex128 spectra)",
        "data": "synthetic: real U(-1,1) field, torch Philox seed 33",
        "config": {"workload": "config3: physical 257x256x256 (n_x=256 Gauss, n_y=n_z=256), nu=dt=1e-3",
                   "l2_policy": "each stage streams >= 135 MB arrays (> L2)"},
        "stages_ms": stages,
        "wall_normal_stages": wall["stages"],
        "roofline": wall["roofline"],
        "gpu_launches": 10 * args.steps,  # per step: 2 x (plane rfft2, wall forward, solve, wall inverse, plane irfft2)
        "solved_unknowns_per_s": unk * args.steps / (total_ms / 1e3),
        "cpu_baseline": cpu, "clocks": clk.summary(),
    }))


def run_c3_slab(args):
    """Config 3 on several ranks: every rank holds its x-planes of the field
    and its folded kx rows of the spectra.  One step =
    the same six stages as run_c3 through distributed.forward_transform_slab /
    inverse_transform_slab, with the kx-row exchange fused into the plane FFT
    kernels over peer memory (distributed.PeerExchange), and the solves of
    the rank's rows.  Strong scaling: the field is fixed, max over ranks.
    SHEN_BENCH_BACKEND=gloo lets several ranks share one GPU (the launcher's
    test; NCCL refuses that) -- not a bench number."""
    import torch
    import torch.distributed as dist

    from paper_1701_03787_b200 import distributed as D
    from paper_1701_03787_b200 import solvers as S
    from paper_1701_03787_b200.matrices import assemble
    from paper_1701_03787_b200.mesh import Space, build_mesh, wavenumber_grid

    rank, world, local = dist_env()
    backend = os.environ.get("SHEN_BENCH_BACKEND", "nccl")
    shared_gpu = backend == "gloo"
    dev = 0 if shared_gpu else local
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group(backend)
    nu, dt = 1e-3, 1e-3
    n_x = int(os.environ.get("SHEN_BENCH_C3_NX", "256"))  # the launcher's test uses a thin mesh
    mesh = build_mesh(n_x, 256, 256, 2 * np.pi, np.pi)
    N = n_x + 1
    mats = assemble(n_x, 0)
    rows = D.kx_rows(mesh.n_y, rank, world)
    z2 = wavenumber_grid(mesh, Space.DIRICHLET).z2()[rows]
    hlu = S.build_helmholtz(mats, nu, dt, z2)
    blu = S.build_biharmonic(mats, nu, dt, z2)
    lo, hi = D.plane_slab(N, rank, world)
    g = torch.Generator(device="cuda").manual_seed(33)
    u = (torch.rand(mesh.shape, generator=g, device="cuda", dtype=torch.float64) * 2 - 1)[lo:hi].contiguous()
    ex = D.PeerExchange(N, mesh.n_y, mesh.n_z)
    out = {}

    def step():
        cd = D.forward_transform_slab(u, mesh, Space.DIRICHLET, exchange=ex)
        xh = hlu.solve(cd)
        out["ud"] = D.inverse_transform_slab(xh, mesh, Space.DIRICHLET, exchange=ex)
        cb = D.forward_transform_slab(u, mesh, Space.BIHARMONIC, exchange=ex)
        xb = blu.solve(cb)
        out["ub"] = D.inverse_transform_slab(xb, mesh, Space.BIHARMONIC, exchange=ex)

    warm = max(args.warmup, 3)
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    with ClockSampler(dev) as clk:
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(args.steps):
            step()
        t1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    total_ms = float(ms.item())
    if rank == 0:
        B = mesh.n_y * (mesh.n_z // 2 + 1)
        print(json.dumps({
            "metric": "config-3 steps/s (fwd transform + solve + inverse, Dirichlet/Helmholtz and biharmonic)",
            "value": args.steps / (total_ms / 1e3), "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": warm, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64 (real field, complex128 spectra)",
            "data": "synthetic: real U(-1,1) field, torch Philox seed 33",
            "config": {"workload": f"config3: physical {N}x256x256 (n_x={n_x} Gauss, n_y=n_z=256), nu=dt=1e-3",
                       "parallelism": f"x-plane slabs / folded kx-row slabs x{world}, exchange fused into the plane "
                                      "FFT kernels (peer memory)" + (", ranks share one GPU (gloo)" if shared_gpu else ""),
                       "l2_policy": "each stage streams arrays larger than L2 at n_x = 256"},
            "solved_unknowns_per_s": (mats.n_dir + mats.n_bih) * B * args.steps / (total_ms / 1e3),
            "gpu_launches": 10 * args.steps, "e2e": None, "clocks": clk.summary()}))
    dist.barrier()
    del ex
    dist.destroy_process_group()


def c3_wall_stages(mesh, u, B):
    """The wall-normal stages of config 3 on their own (the fused
    shen_wall.cu kernels behind transforms.wall_forward / wall_inverse), each
    timed with CUDA events over 10 launches, and their HBM roofline:
    algorithmic bytes = (rows in + rows out) x L lines x 16 B per launch
    (complex128 Fourier lines in, coefficients out, or the reverse)."""
    import torch

    from paper_1701_03787_b200 import transforms as T
    from paper_1701_03787_b200.mesh import family_code

    peak, peak_src = measured_peak()
    fam = family_code(mesh.family)
    lines = torch.fft.rfft2(u, dim=(1, 2)).contiguous().view(mesh.n_x + 1, -1)
    L = lines.shape[1]
    res = {}
    for sp, name in ((1, "dirichlet"), (2, "biharmonic")):
        n = mesh.n_x - 1 if sp == 1 else mesh.n_x - 3
        coef = T.wall_forward(lines, mesh.n_x, fam, sp, True)
        for kind, fn, rows in (("forward", lambda: T.wall_forward(lines, mesh.n_x, fam, sp, True), n + mesh.n_x + 1),
                               ("inverse", lambda: T.wall_inverse(coef, mesh.n_x, fam, sp, mesh.n_y * mesh.n_z),
                                n + mesh.n_x + 1)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            byts = rows * L * 16
            res[f"{kind}_{name}"] = {"ms": ms, "bytes": byts, "GBps_alg": byts / (ms * 1e6), "frac": byts / (ms * 1e6) / peak}
    # the periodic plane FFTs (csrc/shen_plane_fft.cu): 257 planes, real 256 x 256 <-> 256 x 129 complex
    planes = mesh.n_x + 1
    pbytes = planes * mesh.n_y * (mesh.n_z * 8 + (mesh.n_z // 2 + 1) * 16)
    spec = T.plane_rfft2(u)
    for kind, fn in (("plane_rfft2", lambda: T.plane_rfft2(u)),
                     ("plane_irfft2", lambda: T.plane_irfft2(spec, mesh.n_y, mesh.n_z, "forward"))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res[kind] = {"ms": ms, "bytes": pbytes, "GBps_alg": pbytes / (ms * 1e6), "frac": pbytes / (ms * 1e6) / peak}
    dom = max((k for k in res if not k.startswith("plane")), key=lambda k: res[k]["ms"])
    # DRAM bytes per launch of that kernel from the committed ncu launch list
    # (profiles/r02/c3_launches_summary.json, cold-cache serialised launches)
    traffic, tsrc = None, None
    try:
        summ = json.load(open(os.path.join(ROOT, "profiles", "r02", "c3_launches_summary.json")))
        want = "wall_forward_kernel" if dom.startswith("forward") else "wall_inverse_kernel"
        ent = [e for e in summ if want in e["kernel"]]
        if ent:
            traffic = float(ent[0]["dram_bytes_per_launch"])
            tsrc = f"ncu launch list, profiles/r02/c3_launches_summary.json ({want}, mean over the step's launches)"
    except Exception:
        pass
    roof = {"bound": "hbm", "kernel": f"shen_wall {dom} (fused DCT + stencil + mass solve)", "achieved": res[dom]["GBps_alg"],
            "peak": peak, "unit": "GB/s", "frac": res[dom]["frac"], "traffic": traffic, "traffic_source": tsrc,
            "peak_source": peak_src, "algorithmic_bytes": "(rows in + rows out) x 33,024 lines x 16 B per launch"}
    return {"stages": res, "roofline": roof}


def cpu_c3():
    """Oracle port of the same step (numpy/scipy pocketfft + LAPACK, reference
    arithmetic) on a bounded sample: the full 257-point wall-normal direction
    on a 256 x 32 plane (1/8 of config 3), 1 thread; reported per full step."""
    from oracle import shen_oracle as O
    from paper_1701_03787_b200.matrices import assemble
    from paper_1701_03787_b200.mesh import Space, build_mesh, wavenumber_grid

    nu, dt = 1e-3, 1e-3
    mesh = build_mesh(256, 256, 32, 2 * np.pi, np.pi)
    mats = assemble(256, 0)
    z2 = wavenumber_grid(mesh, Space.DIRICHLET).z2()
    u = np.random.default_rng(33).uniform(-1, 1, mesh.shape)
    hf = O.helmholtz_factor(mats, nu, dt, z2)
    bf = O.biharmonic_factor(mats, nu, dt, z2)
    t0 = time.perf_counter()
    cd = O.forward_transform(u, 1, False, mats)
    xd = O.helmholtz_solve(hf, cd)
    O.inverse_transform(xd, 1, False, 256, 256, 32)
    cb = O.forward_transform(u, 2, False, mats)
    xb = O.biharmonic_solve(bf, cb)
    O.inverse_transform(xb, 2, False, 256, 256, 32)
    t = time.perf_counter() - t0
    full = t * (256 // 2 + 1) / (32 // 2 + 1)
    return {"value": 1.0 / full, "unit": "steps/s", "cores": 1, "kind": "port",
            "sample": f"257 x 256 x 32 plane ({t:.2f} s), scaled by kz columns 129/17 to the full step"}


# ======================================================================= full time step

def run_step(args):
    """One reference time step (ChannelStepper.step, stepper.py:286-346)
    composed of the device pieces (stepper.DeviceStepper) on the config-3 mesh
    (n_x = 256, 256 x 256), fixed-beta forcing, nu = 1/2000, dt = 1e-4;
    random spectral state (torch Philox).  CPU baseline: the oracle's
    restatement of the same step (nonlinear term, RHS, solves, recovery) once
    on one core."""
    import torch

    from paper_1701_03787_b200.checkpoint import FlowState
    from paper_1701_03787_b200.mesh import Space, build_mesh, wavenumber_grid
    from paper_1701_03787_b200.stepper import DeviceStepper
    from paper_1701_03787_b200.transforms import SpectralField

    rank, world, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)

    class Cfg:
        nu, dt, forcing, beta, target_flux, dealias = 1 / 2000, 1e-4, "fixed-beta", 0.01, 0.0, True

    mesh = build_mesh(256, 256, 256, 2 * np.pi, np.pi)
    t_build = time.perf_counter()
    stp = DeviceStepper(mesh, Cfg)
    t_build = time.perf_counter() - t_build
    gd, gb = wavenumber_grid(mesh, Space.DIRICHLET), wavenumber_grid(mesh, Space.BIHARMONIC)
    gen = torch.Generator(device="cuda").manual_seed(7)

    def field(grid):
        shp = (grid.n_modes,) + mesh.spectral_shape_yz
        return SpectralField(torch.randn(shp, dtype=torch.complex128, device="cuda", generator=gen), grid, mesh)

    state = FlowState(field(gb), field(gd), field(gd), field(gd), tuple(field(gd) for _ in range(3)),
                      tuple(field(gd) for _ in range(3)), 0.01, 0.0, 0)
    # warm-up advances the state exactly like the timed loop (same allocation
    # pattern: each step holds the previous state's nonlinear term)
    s = state
    for _ in range(max(args.warmup, 3)):
        s = stp.step(s)
    torch.cuda.synchronize()
    # The eager step is ~150 launches from Python, close to host-bound: a host
    # hiccup inside one short timed block shows up whole.  Time 5 blocks of K
    # steps and report the median block (all five in "blocks_ms_per_step").
    blocks = []
    with ClockSampler(local) as clk:
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                s = stp.step(s)
            e1.record()
            torch.cuda.synchronize()
            blocks.append(e0.elapsed_time(e1) / args.steps)
    ms = float(np.median(blocks))
    cpu = None if args.no_cpu else cpu_step(stp, state)
    print(json.dumps({
        "metric": "time steps/s (reference ChannelStepper.step composed of the device kernels)",
        "value": 1e3 / ms, "unit": "steps/s", "n_gpus": 1, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": ms, "higher_is_better": True, "scaling": "none", "vs_baseline": None,
        "dtype": "f64 (complex128 spectra)", "data": "synthetic: random spectral state (torch Philox seed 7)",
        "config": {"workload": "stepper step on the config-3 mesh: n_x=256 (Gauss), 256x256, nu=1/2000, "
                               "dt=1e-4, fixed beta; 8 inverse + 3 forward transforms, 2 RHS, 2 batched solves, "
                               "velocity recovery, mean-flow solve",
                   "l2_policy": "every field 135 MB (> L2)"},
        "blocks_ms_per_step": blocks, "timing": "median of 5 blocks of `steps` eager steps (CUDA events)",
        "build_s": t_build, "cpu_baseline": cpu, "clocks": clk.summary()}))


def cpu_step(stp, state):
    """The oracle's restatement of the same step, once, one core."""
    from oracle import shen_oracle as O

    mats, mesh = stp.mats, stp.mesh
    h = lambda f: f.data.cpu().numpy()  # noqa: E731
    u, v, w, g = h(state.u_hat), h(state.v_hat), h(state.w_hat), h(state.g_hat)
    hc = [h(x) for x in state.h_curr]
    nu, dt = stp.config.nu, stp.config.dt
    hf = O.helmholtz_factor(mats, nu, dt, stp.z2)
    bf = O.biharmonic_factor(mats, nu, dt, stp.z2)
    t0 = time.perf_counter()
    h_new = O.compute_nonlinear(mats, False, mesh.n_y, mesh.n_z, stp.m, stp.n, stp.mask, u, v, w, g)
    hab = O.ab2(h_new, hc)
    u_new = O.biharmonic_solve(bf, O.assemble_rhs_u(mats, nu, dt, stp.z2, stp.m, stp.n, u, hab))
    g_new = O.helmholtz_solve(hf, O.assemble_rhs_g(mats, nu, dt, stp.z2, stp.m, stp.n, g, hab))
    O.recover_velocity(mats, stp.z2, stp.m, stp.n, u_new, g_new)
    t = time.perf_counter() - t0
    return {"value": 1.0 / t, "unit": "steps/s", "cores": 1, "kind": "port",
            "sample": f"one full step on the same mesh ({t:.1f} s; LU prebuilt, mean-flow solve omitted)"}


# ======================================================================= reference arm

_REF_CACHE = {}


def _ref_worker(task):
    """One pool task: the oracle port's solve of a 2-kx-row slab.  LU objects
    and right-hand sides are built on first use and cached in the
    (persistent) worker process, so the timed steps contain only the solves
    -- the same split as the B200 arm (LU built once before timing)."""
    import os as _os

    _os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import shen_oracle as O
    from paper_1701_03787_b200.matrices import assemble
    from paper_1701_03787_b200.mesh import channel_z2

    cfg, lo, hi, seed = task
    # tasks are equal-sized slabs; a worker keeps the first slab it was given
    # (pool scheduling does not pin tasks to workers) and solves it every step
    key = cfg
    if key not in _REF_CACHE:
        name, n_x, n_y, n_z, nu, dt = workload(cfg)
        mats = assemble(n_x, 0)
        z2 = np.ascontiguousarray(channel_z2(n_y, n_z)[lo:hi])
        rng = np.random.default_rng(seed)
        fh = rng.standard_normal((mats.n_dir,) + z2.shape) + 1j * rng.standard_normal((mats.n_dir,) + z2.shape)
        fb = rng.standard_normal((mats.n_bih,) + z2.shape) + 1j * rng.standard_normal((mats.n_bih,) + z2.shape)
        _REF_CACHE[key] = (O.helmholtz_factor(mats, nu, dt, z2), O.biharmonic_factor(mats, nu, dt, z2), fh, fb,
                           (mats.n_dir + mats.n_bih) * z2.size)
    hf, bf, fh, fb, unk = _REF_CACHE[key]
    t0 = time.perf_counter()
    O.helmholtz_solve(hf, fh)
    O.biharmonic_solve(bf, fb)
    return unk, time.perf_counter() - t0


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp

    name, n_x, n_y, n_z, nu, dt = workload(args.config)
    cores = os.cpu_count() or 1
    rows_per_task = 2
    ctx = mp.get_context("spawn")
    results = []
    with ctx.Pool(cores) as pool:
        tasks = [(args.config, (r * rows_per_task) % n_y, (r * rows_per_task) % n_y + rows_per_task, r)
                 for r in range(cores)]
        for _ in range(max(args.warmup, 1)):  # first pass builds and caches each worker's LU + RHS
            pool.map(_ref_worker, tasks, chunksize=1)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            results.extend(pool.map(_ref_worker, tasks, chunksize=1))
        wall = time.perf_counter() - t0
    unk = sum(r[0] for r in results)
    value = unk / wall
    print(json.dumps({
        "impl": "reference",
        "metric": "solved unknowns/s (batched fp64 Helmholtz+biharmonic); % of HBM roofline",
        "value": value, "unit": "unknowns/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 (complex128)",
        "data": "synthetic complex128 N(0,1)",
        "config": {"workload": name, "sample_per_step": f"{cores} x {rows_per_task} kx rows x 1025 systems"},
        "cpu_baseline": {"value": value, "unit": "unknowns/s", "cores": cores, "kind": "port",
                         "sample": f"each step: {cores} processes x {rows_per_task} kx rows of {name}; "
                                   "oracle port of chebchan solve (numpy, identical arithmetic), LU prebuilt"},
        "e2e": {"value": value, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def spawn_ranks(n: int) -> int:
    """``bench.py --gpus N`` without torchrun: start one process per GPU
    (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR=127.0.0.1 / MASTER_PORT in
    the environment, NCCL_DEBUG=INFO unless set, so the NCCL init lines on
    stderr show nranks), rank 0 prints the JSON line.  Returns the worst exit
    code."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        env.setdefault("NCCL_DEBUG", "INFO")
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    codes = [p.wait() for p in procs]
    return max(abs(c) for c in codes)


if __name__ == "__main__":
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and a.impl != "reference":
        sys.exit(spawn_ranks(a.gpus))
    if "WORLD_SIZE" in os.environ and a.gpus != int(os.environ["WORLD_SIZE"]):
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}; using WORLD_SIZE",
              file=sys.stderr)
    if a.dry_run:
        run_dry(a)
    elif a.impl == "reference":
        run_reference(a)
    elif a.config == "c3":
        run_c3(a)
    elif a.config == "step":
        run_step(a)
    else:
        run_b200(a)
