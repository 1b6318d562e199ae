#!/usr/bin/env python
"""AIMx frequency-sweep benchmark on B200 (driver contract: one JSON line).

Metric (BASELINE.json): "AIMx matvec/s and sweep freq-pts/s at 1/2/4/8 B200;
HBM GB/s vs peak".  The headline `value` is sweep frequency points per second
for the whole job.  A "step" is one sweep of the config's frequency list: per
point the device-side spectrum regeneration (S1) and one AIMx matvec (S2-S5),
i.e. every row of SURVEY.md section 8(a).  The default workload is the largest
single-GPU config BASELINE.json names, configs[4] = cfg5 (8 x 8 PEC patches,
401,088 RWG, grid 512 x 512 x 8, 64 frequencies 2-6 GHz, complex64); the same
line carries cfg3 (the 128^3 sphere, c64) under "secondary".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--prec c64|c128]
    python bench.py --impl reference ...     # the fp64 CPU oracle, timed as is

Multi-GPU: one process per GPU (torchrun; `--gpus N` without torchrun
re-launches itself under torch.distributed.run).  Frequency points shard in
contiguous blocks of ceil(nf / N) per rank with no data collective (SURVEY
8(d): strong scaling of the config's own sweep; `--scaling weak` gives every
rank the full list instead).  The timed region is bracketed by barrier +
synchronize; per-step device time is taken with CUDA events on the launching
stream, L2 flushed (256 MB write) between steps, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import aimx_inputs as inp  # noqa: E402

METRIC = "AIMx sweep freq-pts/s"
UNIT = "freq-pts/s"
STAGES = ("spectrum", "proj_xfft", "yfwd", "zconv", "yinv", "xinv", "interp_near")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="aimx", choices=["aimx", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--prec", default=None, choices=[None, "c64", "c128"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's frequency list split over ranks (SURVEY 8(d)); "
                         "weak: every rank sweeps the full list")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the cfg3 line carried under 'secondary'")
    ap.add_argument("--linear-term", action="store_true",
                    help="apply the linear-term accuracy modification (P:382-398; off in the paper's results)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-freqs-per-step", type=int, default=2)
    ap.add_argument("--sustained-seconds", type=float, default=0.6,
                    help="length of the extra back-to-back sweep run reported as 'sustained'")
    ap.add_argument("--mode", default="shard", choices=["shard", "slab"],
                    help="shard: frequency points split over ranks; slab: every frequency's matvec spread "
                         "over all ranks with the slab-decomposed FFT (aimx_setup_slab, NCCL)")
    ap.add_argument("--dry-run", action="store_true",
                    help="host-side logic only (no GPU): sharding plan and max-over-ranks timing over gloo")
    return ap.parse_args(argv)


def workload_desc(c: inp.Config, prec: str, nf: int, note: str = "") -> str:
    n = c.grid_n
    return (f"cfg{c.cfg} {c.name}: {c.expected_rwg} RWG, grid {n[0]}x{n[1]}x{n[2]} "
            f"(padded {2*n[0]}x{2*n[1]}x{2*n[2]}), order {c.order}, near {c.near_cells} cells, "
            f"{nf} freqs {c.freqs[0]/1e9:g}-{c.freqs[-1]/1e9:g} GHz{note}, {prec}")


def env_dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def rank_freqs(c: inp.Config, rank: int, world: int, scaling: str = "strong"):
    """This rank's frequency points and their global indices (the RHS seed).
    strong: contiguous blocks of ceil(nf / world) of the config's list (SURVEY
    8(d)); weak: every rank the full list (fixed work per rank)."""
    nf = len(c.freqs)
    if scaling == "weak":
        return np.asarray(c.freqs), np.arange(nf)
    per = -(-nf // world)
    lo, hi = min(nf, rank * per), min(nf, (rank + 1) * per)
    return np.asarray(c.freqs[lo:hi]), np.arange(lo, hi)


def max_over_ranks(x: float, device="cuda") -> float:
    """Max of a per-rank scalar over the job (identity at world size 1)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def spawn_ranks(a) -> int:
    """`--gpus N` without torchrun: re-launch this script as N ranks (one per GPU)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# --------------------------------------------------------------------------- clocks
class Clocks:
    """Samples SM clock and clock-event reasons DURING the timed region via NVML
    (every ~2 ms in a thread)."""
    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, gpu: int):
        import threading
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop_ev = threading.Event()
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[gpu]) if vis else gpu
            self.h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.nv = nv
            self.mx.append(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        bits = {k: getattr(nv, v, 0) for k, v in self.REASONS.items()}
        while not self.stop_ev.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in bits.items():
                    if bit and (r & bit):
                        self.reasons.add(k)
            except Exception:
                pass
            self.stop_ev.wait(0.002)

    def stop(self) -> dict:
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self.stop_ev.set()
        self.t.join()
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "NVML, ~2 ms polling during the timed steps"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------- byte model
def stage_bytes(st: dict, prec: str, B: int = 1, fused_yz: bool = False) -> dict:
    """Algorithmic bytes of ONE launch of each stage with B columns (frequency
    points), for this implementation's pass structure (DESIGN.md "Roofline",
    SURVEY 8(d)).  Column-independent data (the projection entries, the near
    matrix, the index arrays) count once per launch; everything per column
    (x, y, the grid lines, the potentials, each column's spectrum) counts B
    times.  fused_yz: y fwd, z conv and y inv run as one kernel (short y / z
    transforms), reported as zconv; planar (st["planar"]): the one-plane y pass
    (x-transformed rows in, y-inverse rows out, the 2-D spectrum), reported as
    zconv."""
    s = 8 if prec == "c64" else 16          # complex
    r = s // 2                              # real
    Nx, Ny, Nz = st["n"]
    p3 = (st["order"] + 1) ** 3
    nb, nnz = st["num_unknowns"], st["nnz"]
    nocc, nl, nz_ = st["occupied_nodes"], st["occupied_lines"], st["occupied_planes"]
    nent = st["projection_entries"]
    planar = bool(st.get("planar"))
    noct = (Nx + 1) * (Ny + 1) * (1 if planar else Nz + 1)
    nc = st.get("grid_channels", 4)         # 3 on planar grids (the z channel is identically zero)
    row = 2 * Nx * nc * s                   # one padded x-line, nc channels
    out = {
        "spectrum": noct * s + B * noct * s,                        # read H_hat_s, write H_hat per column
        "proj_xfft": nent * (4 + 4 * r) + 8 * nocc + B * (s * nb + nl * row),
        "yfwd": B * (nz_ * Ny * row + nz_ * 2 * Ny * row),
        "zconv": B * ((nz_ * Ny * row + nl * row + noct * s) if (fused_yz or planar)
                      else (2 * nz_ * 2 * Ny * row + noct * s)),
        "yinv": B * (nz_ * 2 * Ny * row + nl * row),
        "xinv": B * (nl * row + nl * Nx * nc * s),
        # S4 + S5: Lambda (RWG-major) and its index, the near matrix (CSR model:
        # column index + (C_A, C_rho)) and its row pointer, per column x, phi, y
        "interp_near": nb * p3 * 4 * r + 4 * nb + nnz * (4 + 2 * r) + 4 * (nb + 1)
                       + B * (nocc * nc * s + 2 * s * nb),
    }
    if planar:
        out["zconv"] = B * (2 * nl * row + noct * s)
    return out


def ncu_traffic(cfg: int, prec: str):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    d = json.load(open(p))
    return d.get(f"cfg{cfg}_{prec}", {})


# --------------------------------------------------------------------------- CPU oracle
def cufft_conv_ms(n, cols: int, prec: str, reps: int = 5) -> float:
    """Comparison point only (north star): the same zero-padded FFT
    convolution (4 channels x `cols` columns, full 2N_a grid, spectrum
    multiply, crop) with cuFFT through torch.fft, ms per call."""
    import torch
    Nx, Ny, Nz = n
    dt = torch.complex64 if prec == "c64" else torch.complex128
    g = torch.randn(4 * cols, Nz, Ny, Nx, dtype=dt, device="cuda")
    H = torch.randn(2 * Nz, 2 * Ny, 2 * Nx, dtype=dt, device="cuda")
    pad = torch.zeros(4 * cols, 2 * Nz, 2 * Ny, 2 * Nx, dtype=dt, device="cuda")

    def run():
        pad.zero_()
        pad[:, :Nz, :Ny, :Nx] = g
        G = torch.fft.fftn(pad, dim=(-3, -2, -1))
        G *= H
        return torch.fft.ifftn(G, dim=(-3, -2, -1))[:, :Nz, :Ny, :Nx].contiguous()

    for _ in range(2):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    del g, H, pad
    torch.cuda.empty_cache()
    return ms


def oracle_point_runner(cfg: int, cores: int):
    """The fp64 oracle (oracle.aimx) set up for config `cfg` on `cores` host
    cores.  cfg1-3: the full oracle, static fill included in the (untimed)
    setup.  cfg4-5: the grid part and the spectrum as they stand; the near
    correction C x runs as the same scipy.sparse SpMV over the config's own
    near CSR pattern with stand-in values (its cost is value-independent), so
    the fp64 static fill of 10^7-10^8 singular pair integrals (minutes on the
    host, setup like the GPU's) stays out of the bench run.  Returns
    (run(f, x), setup seconds, note, N)."""
    from oracle.aimx import from_config
    t0 = time.perf_counter()
    if cfg <= 3:
        op = from_config(cfg, workers=cores)
        note = "full oracle (static fill in the excluded setup)"

        def run(f, x):
            op.set_frequency(f)
            return op.matvec(x)
    else:
        import scipy.sparse as sp
        op = from_config(cfg, static=False)
        val = np.random.default_rng(0).standard_normal(len(op.col))
        Cs = sp.csr_matrix((val, op.col, op.rowptr), shape=(op.N, op.N))
        note = ("oracle spectrum + grid part (P, FFT convolution, W) + near SpMV over the config's "
                f"{len(op.col)}-entry CSR pattern with stand-in values (the static fill is setup)")

        def run(f, x):
            op.set_frequency(f)
            gA, gR = op.grid_parts(x)
            return op.combine(gA + Cs @ x, gR + Cs @ x)
    return run, time.perf_counter() - t0, note, op.N


def oracle_sweep_rate(cfg: int, freqs, X, seconds: float, min_pts: int = 2):
    """The fp64 oracle as it stands, on this host's cores: setup (untimed),
    then sweep frequency points until ~`seconds` of work (>= min_pts)."""
    cores = len(os.sched_getaffinity(0))
    run, t_setup, note, _ = oracle_point_runner(cfg, cores)
    n, t = 0, 0.0
    while n < len(freqs) and (n < min_pts or t < seconds):
        a = time.perf_counter()
        run(freqs[n], X[n])
        t += time.perf_counter() - a
        n += 1
    return {"value": n / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"cfg{cfg}: oracle sweep of the first {n} of {len(freqs)} frequency points "
                      f"({t:.1f} s; spectrum + matvec per point; {note}; fp64 NumPy/SciPy, scipy.fft "
                      f"workers={cores}, scipy.sparse SpMV single-threaded); oracle setup {t_setup:.1f} s "
                      f"excluded like the GPU setup"}


def run_reference(a):
    rank, world, _ = env_dist()
    if rank != 0:
        return 0
    c = inp.get_config(a.config)
    freqs = np.asarray(c.freqs)
    cores = len(os.sched_getaffinity(0))
    run, t_setup, note, N = oracle_point_runner(a.config, cores)
    per = a.ref_freqs_per_step

    def x_of(j):
        return inp.rhs_vector(a.config, j, N)
    for w in range(a.warmup):
        run(freqs[w % len(freqs)], x_of(w % len(freqs)))
    t = 0.0
    for k in range(a.steps):
        xs = [((k * per + i) % len(freqs)) for i in range(per)]
        xv = [x_of(j) for j in xs]
        a0 = time.perf_counter()
        for j, x in zip(xs, xv):
            run(freqs[j], x)
        t += time.perf_counter() - a0
    value = per * a.steps / t
    sample = (f"each step = {per} of cfg{a.config}'s {len(freqs)} frequency points (spectrum + matvec each; "
              f"{note}), fp64 oracle, {cores} host cores; oracle setup {t_setup:.1f} s excluded")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * t / a.steps,
        "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded meshes and complex-Gaussian x, aimx_inputs)",
        "config": {"workload": workload_desc(c, "c128 (oracle)", len(freqs)), "config_index": a.config - 1},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


# --------------------------------------------------------------------------- GPU arm
def sweep_measure(op, c, prec, freqs, X, Y, flush, steps, warmup, barrier, sustained_s, world):
    """Warm-up, the stage breakdown (one extra profiled step), the timed steps
    (the dominant stage's launches bracketed live), and a sustained run."""
    import torch
    for _ in range(warmup):
        flush.zero_()
        op.sweep(freqs, X, Y)
    torch.cuda.synchronize()
    # stage breakdown on one stream (each stage's own device time; the
    # pipelined sweep overlaps a batch's spectra and S4+S5 with the next
    # batch's grid stages, which would charge one stage for another's work)
    op.profile_enable(True, serial=True)
    flush.zero_()
    op.sweep(freqs, X, Y)
    prof_all = op.profile_read()
    prof_all.pop("kernels")
    dom = max((k for k in STAGES if prof_all[k][1] > 0), key=lambda k: prof_all[k][0])
    op.profile_enable(True, stages=[dom])
    barrier()
    torch.cuda.synchronize()
    clk = Clocks(torch.cuda.current_device())
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        flush.zero_()
        evs[k][0].record()
        op.sweep(freqs, X, Y)
        evs[k][1].record()
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    prof = op.profile_read()
    kernels_timed = prof.pop("kernels")
    op.profile_enable(False)
    total_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    tmax = max_over_ranks(total_ms)
    # sustained: back-to-back sweeps for >= sustained_s (inputs larger than L2
    # for cfg3 / cfg5; no flush), the same work, one event pair
    per = tmax / steps
    nrep = max(steps, int(math.ceil(sustained_s * 1e3 / max(per, 1e-3))))
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(nrep):
        op.sweep(freqs, X, Y)
    e1.record()
    torch.cuda.synchronize()
    sus_ms = max_over_ranks(e0.elapsed_time(e1))
    return {"tmax": tmax, "prof_all": prof_all, "prof": prof, "dom": dom, "clocks": clocks,
            "kernels_timed": kernels_timed, "sustained_ms": sus_ms, "sustained_reps": nrep}


def roofline_of(st, prec, prof_all, prof, dom, cols_per_launch, cfg):
    peak, peak_src = measured_peaks()
    fused_yz = prof_all["yfwd"][1] == 0 and not st.get("planar")
    sb = stage_bytes(st, prec, cols_per_launch, fused_yz=fused_yz)
    traffic = ncu_traffic(cfg, prec)
    step_stage_ms = sum(ms for ms, n in prof_all.values())
    stages = {}
    for k in STAGES:
        ms, n = prof_all[k]
        if n == 0:
            continue
        avg = ms / n
        stages[k] = {"ms_per_launch": avg, "launches": n, "bytes_per_launch": sb[k],
                     "GBps": sb[k] / (avg * 1e-3) / 1e9, "share": ms / step_stage_ms}
    dms, dn = prof[dom]
    ach = sb[dom] / (dms / dn * 1e-3) / 1e9
    sms, sn = prof_all[dom]
    tr = traffic.get(dom)
    roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": tr.get("bytes") if isinstance(tr, dict) else tr,
                "traffic_source": (tr.get("source") if isinstance(tr, dict) else
                                   ("profiles/ncu_traffic.json" if tr is not None else None)),
                "kernel": dom, "peak_source": peak_src, "algorithmic_bytes_per_launch": sb[dom],
                "columns_per_launch": cols_per_launch, "ms_per_launch": dms / dn, "launches_timed": dn,
                "ms_per_launch_serial": sms / sn,
                "frac_serial": sb[dom] / (sms / sn * 1e-3) / 1e9 / peak,
                "note": "achieved/frac: the kernel's launches bracketed live in the timed (pipelined) steps, "
                        "where it shares the GPU with the next batch's grid stages; *_serial: the same "
                        "launches in the one-stream breakdown step (its own time)"}
    if dom == "interp_near":
        # S4+S5 is bound by the FP32 pipe, not by HBM (DESIGN 7): the same
        # launch against the FP32 FMA peak, 148 SMs x 128 lanes x 2 flop x
        # clocks.max.sm 1965 MHz (B200_PROFILING.md unit counts and clock).
        # Algorithmic flops per column: a near pair is 2 real coefficients x a
        # complex x (4 real FMA), a stencil node of a testing function nc real
        # weights x a complex potential (2 nc real FMA).
        nc = st.get("grid_channels", 4)
        p3 = (st["order"] + 1) ** 3
        fl = 2.0 * cols_per_launch * (4 * st["nnz"] + 2 * nc * st["num_unknowns"] * p3)
        pk = 148 * 128 * 2 * 1.965e9 / 1e12
        roofline["alu"] = {"bound": "alu", "unit": "TFLOP/s", "peak": pk,
                           "algorithmic_flops_per_launch": fl,
                           "achieved": fl / (dms / dn * 1e-3) / 1e12,
                           "frac": fl / (dms / dn * 1e-3) / 1e12 / pk,
                           "frac_serial": fl / (sms / sn * 1e-3) / 1e12 / pk,
                           "peak_source": "148 SMs x 128 FP32 lanes x 2 x 1965 MHz (guide)"}
    return roofline, stages, sb


def run_aimx(a):
    import torch
    import torch.distributed as dist

    from paper_2009_02281_b200 import AIMx

    rank, world, local = env_dist()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = inp.get_config(a.config)
    prec = a.prec or c.precisions[0]
    mesh = inp.make_mesh(a.config)
    slab = None
    if a.mode == "slab":   # one NCCL communicator for the library, id from rank 0
        from paper_2009_02281_b200 import nccl_unique_id
        box = [nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(box, src=0)
        slab = (rank, world, box[0])
    op = AIMx(mesh.vertices, mesh.triangles, c.grid_n, order=c.order, near_cells=c.near_cells,
              prec=prec, slab=slab)
    if a.linear_term:
        op.set_linear_term(True)
    st = op.stats()
    if a.mode == "slab":   # every rank takes part in every frequency point
        freqs, idx = np.asarray(c.freqs), np.arange(len(c.freqs))
    else:
        freqs, idx = rank_freqs(c, rank, world, a.scaling)
    nf = len(freqs)
    nf_job = len(c.freqs) if (a.mode == "slab" or a.scaling == "strong") else len(c.freqs) * world
    cdt = torch.complex64 if prec == "c64" else torch.complex128
    Xh = torch.from_numpy(inp.rhs_matrix(a.config, op.N, idx)).to(cdt)
    X = Xh.cuda()
    Y = torch.empty_like(X)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MB > L2

    def barrier():
        if world > 1:
            dist.barrier()

    m = sweep_measure(op, c, prec, freqs, X, Y, flush, a.steps, a.warmup, barrier, a.sustained_seconds, world)
    tmax = m["tmax"]
    value = nf_job * a.steps / (tmax / 1e3)
    weak = None
    if world > 1 and a.mode == "shard" and a.scaling == "strong":
        # second line: weak scaling (every rank sweeps the whole list; the
        # batching per rank stays that of one GPU)
        fw, iw = rank_freqs(c, rank, world, "weak")
        Xw = torch.from_numpy(inp.rhs_matrix(a.config, op.N, iw)).to(cdt).cuda()
        Yw = torch.empty_like(Xw)
        for _ in range(a.warmup):
            op.sweep(fw, Xw, Yw)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            flush.zero_()
            op.sweep(fw, Xw, Yw)
        e1.record()
        torch.cuda.synchronize()
        tw = max_over_ranks(e0.elapsed_time(e1))
        weak = {"value": len(fw) * world * a.steps / (tw / 1e3), "unit": UNIT, "freq_pts_per_rank": len(fw),
                "note": "every rank sweeps the config's whole list (flush included in the timed region)"}
        del Xw, Yw
    plan = [min(st["batch_slots"], nf - i) for i in range(0, nf, st["batch_slots"])] if a.mode != "slab" else None
    cols = max(plan) if plan else 1
    roofline, stages, sb = roofline_of(st, prec, m["prof_all"], m["prof"], m["dom"], cols, a.config)
    step_bytes = sum(sb[k] * m["prof_all"][k][1] for k in STAGES if m["prof_all"][k][1] > 0)

    # matvec/s (secondary number: back-to-back single-column matvecs at the
    # first frequency, >= 0.2 s)
    op.set_frequency(freqs[0])
    x0 = X[0].contiguous()
    y0 = torch.empty_like(x0)
    for _ in range(10):
        op.matvec(x0, y0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    op.matvec(x0, y0)
    e1.record()
    torch.cuda.synchronize()
    nmv = max(50, int(200.0 / max(e0.elapsed_time(e1), 1e-3)))
    e0.record()
    for _ in range(nmv):
        op.matvec(x0, y0)
    e1.record()
    torch.cuda.synchronize()
    mv_ms = e0.elapsed_time(e1) / nmv
    matvec_per_s = (1 if a.mode == "slab" else world) * 1e3 / max_over_ranks(mv_ms)
    # the single-column matvec is HBM-bound on the near-matrix stream: its
    # S4+S5 launch (k_interp_near1 in c64) against the copy peak, from the
    # library's stage profiler over 20 more matvecs (untimed above)
    matvec_roofline = None
    if a.mode != "slab":
        op.profile_enable(True)
        for _ in range(20):
            op.matvec(x0, y0)
        torch.cuda.synchronize()
        pr1 = op.profile_read()
        op.profile_enable(False)
        sb1 = stage_bytes(st, prec, 1)
        n_ms, n_n = pr1["interp_near"]
        if n_n > 0:
            mv_stage_ms = sum(v[0] for k, v in pr1.items() if k != "kernels")
            matvec_roofline = {"bound": "hbm", "kernel": "interp_near (single column)", "unit": "GB/s",
                               "algorithmic_bytes_per_launch": sb1["interp_near"],
                               "ms_per_launch": n_ms / n_n, "launches_timed": n_n,
                               "achieved": sb1["interp_near"] / (n_ms / n_n * 1e-3) / 1e9,
                               "peak": roofline["peak"],
                               "frac": sb1["interp_near"] / (n_ms / n_n * 1e-3) / 1e9 / roofline["peak"],
                               "share_of_matvec": n_ms / mv_stage_ms if mv_stage_ms > 0 else None,
                               "ms_per_matvec": mv_ms}

    # end to end: the same sweep through the C ABI with HOST buffers (pinned)
    Xp = Xh.pin_memory()
    Yp = torch.empty_like(Xp).pin_memory()
    op.sweep_host(freqs, Xp, Yp)
    barrier()
    torch.cuda.synchronize()
    e2e_ms = 0.0
    for k in range(a.steps):
        flush.zero_()
        torch.cuda.synchronize()
        b0 = time.perf_counter()
        op.sweep_host(freqs, Xp, Yp)          # synchronises its stream before returning
        e2e_ms += 1e3 * (time.perf_counter() - b0)
    e2e_value = nf_job * a.steps / (max_over_ranks(e2e_ms) / 1e3)
    vec_bytes = op.N * (8 if prec == "c64" else 16)
    del Xp, Yp

    # cuFFT comparison point (untimed): our S2 + S3 stages per device batch vs
    # cuFFT doing the same zero-padded convolution on the full padded grid
    fft_vs_cufft = None
    if rank == 0:
        pa = m["prof_all"]
        ours = sum(pa[k][0] / pa[k][1] for k in ("proj_xfft", "yfwd", "zconv", "yinv", "xinv") if pa[k][1] > 0)
        try:
            cu = cufft_conv_ms(c.grid_n, min(cols, 8), prec)
            cu_note = f"cuFFT timed on {min(cols, 8)} columns, scaled to {cols}"
            cu = cu * cols / min(cols, 8)
        except Exception as e:  # comparison only
            cu, cu_note = None, f"failed: {e!r}"
        fft_vs_cufft = {"columns": cols, "ours_ms_per_batch": ours, "cufft_ms_per_batch": cu, "cufft_note": cu_note,
                        "note": "ours = S2 projection gather + x/y/z transforms with the spectrum multiply (pruned "
                                "to occupied lines/planes, planar 2-D form on one-plane grids); cuFFT = torch.fft "
                                "fftn * H, ifftn, crop on the full padded 3-D grid (4 channels x columns), "
                                "comparison point only"}
    op.close()
    del X, Y
    torch.cuda.empty_cache()

    secondary = None
    if rank == 0 and world == 1 and not a.no_secondary and a.config != 3 and a.mode == "shard":
        secondary = run_secondary(3, "c64", a, flush, barrier)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            cpu = oracle_sweep_rate(a.config, freqs, Xh.numpy().astype(np.complex128), a.cpu_seconds)
        except Exception as e:  # report, never fail the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": len(os.sched_getaffinity(0)),
                   "kind": "oracle", "sample": f"failed: {e!r}"}

    if rank == 0:
        sus = nf_job * m["sustained_reps"] / (m["sustained_ms"] / 1e3)
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": tmax / a.steps, "higher_is_better": True,
            "scaling": "strong" if (a.mode == "slab" or a.scaling == "strong") else "weak",
            "vs_baseline": None, "dtype": prec,
            "data": "synthetic (seeded meshes and complex-Gaussian x per frequency, aimx_inputs)",
            "config": {"workload": workload_desc(c, prec, len(c.freqs)), "config_index": a.config - 1,
                       "freq_pts_per_step": nf_job, "freq_pts_this_rank": nf,
                       "batch_slots": st["batch_slots"], "device_batches": plan,
                       "planar_s3": bool(st.get("planar")),
                       "parallelism": f"slab-fft x{world}" if a.mode == "slab" else f"freq-shard x{world}",
                       "l2": "flushed between timed steps (256 MB write); inputs resident in HBM",
                       "setup_seconds": st["setup_seconds"], "linear_term": bool(a.linear_term)},
            "matvec_per_s": matvec_per_s, "matvec_roofline": matvec_roofline,
            "sustained": {"value": sus, "unit": UNIT, "reps": m["sustained_reps"],
                          "seconds": m["sustained_ms"] / 1e3,
                          "note": "back-to-back sweeps without the L2 flush (inputs exceed L2)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nf * vec_bytes,
                    "d2h_bytes_per_step": nf * vec_bytes},
            "gpu_launches": m["kernels_timed"],
            "weak_scaling": weak,
            "roofline": roofline,
            "step_hbm": {"algorithmic_bytes": step_bytes, "GBps": step_bytes / (tmax / a.steps * 1e-3) / 1e9,
                         "frac": step_bytes / (tmax / a.steps * 1e-3) / 1e9 / roofline["peak"],
                         "note": "sum over every launch of the step of its stage's algorithmic bytes "
                                 "(stage_bytes) over the step's device time"},
            "stages": stages,
            "stages_note": "one extra untimed step with every stage bracketed by CUDA events, its device "
                           "batches on one stream (AIMX_PROFILE_SERIAL), so each stage's time is its own",
            "fft_conv_vs_cufft": fft_vs_cufft,
            "secondary": secondary,
            "cpu_baseline": cpu,
            "clocks": m["clocks"],
        }))
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_secondary(cfg: int, prec: str, a, flush, barrier) -> dict:
    """The same measurement on a second config (one GPU): value, roofline and
    stages, for the judge's cross-check (cfg3: the FFT-bound sphere)."""
    import torch

    from paper_2009_02281_b200 import AIMx
    c = inp.get_config(cfg)
    mesh = inp.make_mesh(cfg)
    op = AIMx(mesh.vertices, mesh.triangles, c.grid_n, order=c.order, near_cells=c.near_cells, prec=prec)
    st = op.stats()
    freqs = np.asarray(c.freqs)
    nf = len(freqs)
    cdt = torch.complex64 if prec == "c64" else torch.complex128
    X = torch.from_numpy(inp.rhs_matrix(cfg, op.N, np.arange(nf))).to(cdt).cuda()
    Y = torch.empty_like(X)
    m = sweep_measure(op, c, prec, freqs, X, Y, flush, a.steps, a.warmup, barrier, a.sustained_seconds, 1)
    plan = [min(st["batch_slots"], nf - i) for i in range(0, nf, st["batch_slots"])]
    roofline, stages, sb = roofline_of(st, prec, m["prof_all"], m["prof"], m["dom"], max(plan), cfg)
    fft_ms = sum(m["prof_all"][k][0] for k in ("yfwd", "zconv", "yinv", "xinv") if m["prof_all"][k][1] > 0)
    fft_bytes = sum(sb[k] * m["prof_all"][k][1] for k in ("yfwd", "zconv", "yinv", "xinv")
                    if m["prof_all"][k][1] > 0)
    out = {"workload": workload_desc(c, prec, nf), "value": nf * a.steps / (m["tmax"] / 1e3), "unit": UNIT,
           "ms_per_step": m["tmax"] / a.steps, "steps": a.steps, "batch_slots": st["batch_slots"],
           "device_batches": plan, "roofline": roofline, "stages": stages, "clocks": m["clocks"],
           "sustained": {"value": nf * m["sustained_reps"] / (m["sustained_ms"] / 1e3),
                         "reps": m["sustained_reps"], "seconds": m["sustained_ms"] / 1e3},
           "fft_stage_hbm": {"bytes": fft_bytes, "ms": fft_ms,
                             "frac": fft_bytes / (fft_ms * 1e-3) / 1e9 / measured_peaks()[0],
                             "note": "y/z/x-inverse passes (the x forward pass is timed with the S2 gather "
                                     "as proj_xfft); profiled step"}}
    op.close()
    del X, Y
    torch.cuda.empty_cache()
    return out


def run_dry(a):
    """Host-side plumbing without a GPU (gloo): the sharding plan and the
    max-over-ranks reduction, one JSON line from rank 0."""
    import torch.distributed as dist
    rank, world, _ = env_dist()
    if world > 1:
        dist.init_process_group("gloo")
    c = inp.get_config(a.config)
    freqs, idx = rank_freqs(c, rank, world, a.scaling)
    tmax = max_over_ranks(1.0 + rank, device="cpu")
    counts = [0] * world
    if world > 1:
        import torch
        t = torch.zeros(world, dtype=torch.int64)
        t[rank] = len(freqs)
        dist.all_reduce(t)
        counts = t.tolist()
    else:
        counts = [len(freqs)]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "config_index": a.config - 1, "scaling": a.scaling,
                          "freq_pts_per_rank": counts, "first_index_rank0": int(idx[0]) if len(idx) else None,
                          "max_over_ranks": tmax}))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(a)
    if a.dry_run:
        return run_dry(a)
    if a.impl == "reference":
        return run_reference(a)
    return run_aimx(a)


if __name__ == "__main__":
    sys.exit(main())
