"""Benchmark of the gradient-decomposition hot path (arXiv 2205.06327) on B200.

A step = one reconstruction iteration ("a cycle through all the probe locations") of the
LT-small-shaped workload (BASELINE.json configs[3]: 1024x1024x4158 synthetic measurements,
1536x1536x100 object) over the fixed 2x4 tile grid (halo N/2, exact window), tiles spread over
the ranks (8/N virtual tiles per GPU): per-probe forward + adjoint gradient + AccBuf scatter-add
+ SGD for every probe, the four APPP passes, the accumulated step.  Total work is fixed as N
grows ("scaling": "strong"); results are bit-identical for every N.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0 (contract in the task statement).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "probe-locations/sec and sec/iteration at 1/2/4/8 B200; % HBM peak"
# the paper's best GD probe-locations/s per workload: small LT 2310 on 462 V100s
# (Table II(a)), large LT 12 600 on 4158 V100s (Table III(a)); other configs
# have no paper number, so their vs_baseline is null
PAPER_BEST = {"lt_small": 2310.0, "lt_large": 12600.0}


def vs_baseline(cfg, value):
    best = PAPER_BEST.get(cfg.name)
    return value / best if best else None


def env_int(k, d):
    return int(os.environ.get(k, d))


def bind_to_gpu_numa(dev):
    """Pin this rank's host threads to the CPUs local to its GPU (NVML), so the pinned host
    buffers of the e2e leg are first-touched on the GPU's NUMA node.  Returns the CPU count or
    None if NVML / the PCI id is unavailable (then nothing changes)."""
    try:
        import pynvml
        import torch
        pr = torch.cuda.get_device_properties(dev)
        bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        pynvml.nvmlInit()
        pynvml.nvmlDeviceSetCpuAffinity(pynvml.nvmlDeviceGetHandleByPciBusId(bus))
        return len(os.sched_getaffinity(0))
    except Exception:
        return None


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[2 + i]
                          and not s[2 + i].startswith("Not")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------
def workload_name(cfg):
    return (f"{cfg.name}: {cfg.n}x{cfg.n}x{cfg.n_probes} measurements, "
            f"{cfg.width}x{cfg.height}x{cfg.slices} object")


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _oracle_probe_worker(args):
    """One probe's forward + adjoint gradient (oracle.probe_grad, float64) on a window of `slices`
    slices: the unit of the CPU baseline.  Inputs are synthetic of the workload's shape (timing is
    data-independent); numpy's FFT is single-threaded, so one worker = one core."""
    n, slices, sigma, c, seed = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import ptycho_oracle as O
    rng = np.random.default_rng(seed)
    probe = synth.probe(n, 25.0)
    vwin = 0.5 * rng.random((slices, n, n))
    amp = np.abs(np.fft.fft2(probe, norm="ortho"))
    t0 = time.perf_counter()
    O.probe_grad(probe, vwin, amp, sigma, c)
    return time.perf_counter() - t0


def cpu_oracle_sample(cfg, workers, slices_per_probe):
    """The float64 oracle, as it stands, on a bounded sample of the workload: `workers` processes
    (one per core) each compute one probe's forward + adjoint over `slices_per_probe` of the S
    slices (the per-probe cost is linear in S, so the sample is slices_per_probe / S probe-locations
    per worker).  Returns (probe-locations/s, wall seconds, sample text)."""
    import multiprocessing as mp
    frac = slices_per_probe / cfg.slices
    jobs = [(cfg.n, slices_per_probe, cfg.sigma, cfg.prop_c, i) for i in range(workers)]
    t0 = time.perf_counter()
    if workers == 1:
        _oracle_probe_worker(jobs[0])
    else:
        with mp.get_context("spawn").Pool(workers) as pool:
            pool.map(_oracle_probe_worker, jobs, chunksize=1)
    dt = time.perf_counter() - t0
    return workers * frac / dt, dt, (f"{workers} x one {cfg.name} probe (N={cfg.n}) forward+adjoint over "
                                     f"{slices_per_probe} of S={cfg.slices} slices (= {frac:g} probe-locations "
                                     f"each), float64, one process per core")


def cpu_workers():
    """All host cores, capped by memory (one N=1024 probe over 25 slices needs ~0.7 GB)."""
    n = os.cpu_count() or 1
    try:
        import psutil
        n = min(n, max(1, int(psutil.virtual_memory().available / 1.5e9)))
    except Exception:
        pass
    return n


def cpu_tiny_iteration():
    """One full Alg. 1 iteration of the tiny config (BASELINE configs[0]) through oracle.reconstruct."""
    from oracle import ptycho_oracle as O
    c = synth.CONFIGS["tiny"]
    probe = synth.probe(c.n, c.defocus_nm)
    vt = synth.volume(0, c.slices, c.height, c.width).astype(np.float64)
    centers = synth.scan_centers(c.height, c.width, c.scan_ny, c.scan_nx)
    full = (0, 0, c.height, c.width)
    amps = [O.farfield_magnitude(probe, O.window(vt, full, tuple(cc), c.n), c.sigma, c.prop_c) for cc in centers]
    d = dict(n=c.n, sigma=c.sigma, prop_c=c.prop_c)
    t0 = time.perf_counter()
    O.reconstruct(0.5 * vt, probe, amps, centers, d, 1, 1, c.halo, 1, alpha=1.0)
    dt = time.perf_counter() - t0
    return {"config": "tiny (64^2 x 16 probes, 128^2 x 4 object, 1 tile)", "sec_per_iteration": dt,
            "probe_locations_per_s": c.n_probes / dt, "cores": 1}


def run_reference(args):
    """--impl reference: the oracle timed on the host cores (rank 0 only)."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    workers = cpu_workers()
    per = 25 if cfg.slices >= 25 else cfg.slices
    for _ in range(args.warmup):
        cpu_oracle_sample(cfg, workers, per)
    vals, times = [], []
    sample = ""
    for _ in range(args.steps):
        v, dt, sample = cpu_oracle_sample(cfg, workers, per)
        vals.append(v)
        times.append(dt)
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "probe-locations/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.median(times) * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": vs_baseline(cfg, value), "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg), "sample": "per step: " + sample},
            "cpu_baseline": {"value": value, "unit": "probe-locations/s", "cores": workers, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": value, "unit": "probe-locations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def interior_run(p, tile, centers, n, h, w, want=4):
    """first local index of `want` consecutive probes of `tile` whose windows lie inside the object"""
    cnt = p.tile_probe_count(tile)
    # tile's own probes in ascending global order = local_probes restricted to the tile
    ids = [i for i in p.local_probes() if _tile_of(p, i, centers)[0] == tile]
    run = 0
    for j, g in enumerate(ids):
        cy, cx = centers[g]
        ok = cy - n // 2 >= 0 and cy + n // 2 <= h and cx - n // 2 >= 0 and cx + n // 2 <= w
        run = run + 1 if ok else 0
        if run == want:
            return j - want + 1
    return 0 if cnt >= want else None


def _tile_of(p, g, centers):
    cy, cx = centers[g]
    for k in range(p.rows * p.cols):
        _, (y0, x0, y1, x1) = p.tile_rect(k)
        if y0 <= cy < y1 and x0 <= cx < x1:
            return k, None
    return -1, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="lt_small")
    ap.add_argument("--grid", default=None, help="tile grid RxC (default: the config's, 2x4)")
    ap.add_argument("--halo", type=int, default=None,
                    help="halo width (default N/2 = exact window; the paper's circle halo is 60)")
    ap.add_argument("--stash-free", action="store_true",
                    help="stash-free adjoint (PTYCHO_F_STASH_FREE): phi_s recomputed, 2-slice stash")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-async", choices=["auto", "on", "off"], default="auto",
                    help="e2e: PTYCHO_AMP_ASYNC load overlapping the chains; auto = on (with the e2e "
                         "warm-up, interleaved A/B: N=1 +1.2 %%, N=2 +1.2 %%, "
                         "profiles/round2/e2e_async_ab_after_warmup.txt)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist
    from paper_2205_06327_b200.ptycho import Ptycho, PTYCHO_F_STASH_FREE, PTYCHO_AMP_ASYNC

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local_rank)
    numa_cpus = bind_to_gpu_numa(local_rank) if world > 1 else None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    cfg = synth.CONFIGS[args.config]
    R, C = (int(v) for v in args.grid.split("x")) if args.grid else cfg.grid
    ntiles = R * C
    owner = [k * world // ntiles for k in range(ntiles)]
    nid = None
    if world > 1:
        obj = [Ptycho.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    n, S, H, W = cfg.n, cfg.slices, cfg.height, cfg.width
    alpha = 0.5
    stream = torch.cuda.Stream(local_rank)
    p = Ptycho(n, S, H, W, cfg.sigma, cfg.prop_c, alpha=alpha, device=local_rank, stream=stream.cuda_stream,
               flags=PTYCHO_F_STASH_FREE if args.stash_free else 0)
    halo = n // 2 if args.halo is None else args.halo
    p.set_tiles(R, C, halo, owner, nid, rank, world)
    centers = synth.scan_centers(H, W, cfg.scan_ny, cfg.scan_nx)
    p.set_scan(centers)
    ws = p.allocate_workspace()
    probe = synth.probe(n, cfg.defocus_nm)
    p.set_probe(probe.astype(np.complex64))
    vt = synth.volume(0, S, H, W)
    p.set_volume(vt)
    p.simulate_measurements()          # a_i = |G(p_i, V_true)| on the device
    p.set_volume(None)                 # V_0 = 0
    p.synchronize()
    nloc = len(p.local_probes())

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        p.iterate()
    barrier()
    l0 = p.kernel_launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local_rank) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            p.iterate()
        e1.record(stream)
        p.synchronize()
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    launches = p.kernel_launches() - l0
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        lt = torch.tensor([launches], dtype=torch.int64, device="cuda")
        dist.all_reduce(lt)
        launches = int(lt.item())
    value = cfg.n_probes / (ms / 1e3)
    loss = p.iterate(want_loss=True)   # F(V) after K+W+1 iterations (untimed; sanity)

    # ---- APPP exchange alone (N > 1): the four passes over all S slices, CUDA events on the
    # context stream, max over ranks; bytes = cross-rank hop regions x S x 4 B (NVLink roofline)
    appp = None
    if world > 1:
        from paper_2205_06327_b200.ptycho import appp_schedule
        sched = appp_schedule(H, W, R, C, halo)
        xbytes = sum((y1 - y0) * (x1 - x0) * S * 4 for (a, b, y0, y1, x0, x1, _) in sched
                     if owner[a] != owner[b] and y1 > y0 and x1 > x0)
        # bytes each rank receives over NVLink in one call (its hops run in order on its stream):
        # the busiest receiver's bytes / call time = the rate of an active link
        recv = [0] * world
        for (a, b, y0, y1, x0, x1, _) in sched:
            if owner[a] != owner[b] and y1 > y0 and x1 > x0:
                recv[owner[b]] += (y1 - y0) * (x1 - x0) * S * 4
        for _ in range(2):
            p.appp_passes()
        barrier()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(5):
            p.appp_passes()
        a1.record(stream)
        barrier()
        t = torch.tensor([a0.elapsed_time(a1) / 5], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ams = float(t.item())
        appp = {"transport": p.appp_transport(), "ms_per_call": ams, "cross_rank_bytes": xbytes,
                "achieved_gbs_per_gpu": xbytes / world / (ams * 1e6), "nvlink_peak_gbs_per_gpu": 900.0,
                "busiest_receiver_bytes": max(recv), "achieved_gbs_busiest_receiver": max(recv) / (ams * 1e6),
                "frac_of_nvlink_busiest_receiver": max(recv) / (ams * 1e6) / 900.0,
                "note": "not pipelined behind the backward here; in ptycho_iterate the slabs overlap it"}

    # ---- roofline of the dominant kernel (backward middle pass), CUDA events on its stream
    peak, peak_kind = hbm_peak()
    my_tiles = [k for k in range(ntiles) if owner[k] == rank]
    tile = my_tiles[len(my_tiles) // 2]
    j0 = interior_run(p, tile, centers, n, H, W)
    prof = p.profile_chain(tile, j0 or 0, 4) if j0 is not None else {}
    n2 = n * n
    bwd = prof.get("bwd_mid", (0.0, 0))
    fwd = prof.get("fwd_mid", (0.0, 0))
    chain_ms = sum(v[0] for v in prof.values())
    t_bwd = bwd[0] / max(bwd[1], 1) * 1e-3
    t_fwd = fwd[0] / max(fwd[1], 1) * 1e-3
    # compulsory (algorithmic) HBM bytes of one backward middle pass = V read-modify-write
    # 8N^2 + AccBuf read-modify-write 8N^2 = 16N^2; the stash read (8N^2) is a design byte (the
    # stash-free adjoint removes it), reported beside it as "design"
    bytes_bwd = 16 * n2
    bytes_bwd_design = 24 * n2
    bytes_fwd = 4 * n2    # V read (compulsory); + stash write 8N^2 = 12N^2 design
    # In the timed region the tile chains run as CUDA graphs with programmatic dependent launch
    # (and up to 8 tiles concurrently), so a launch's in-step duration is the step time the
    # kernel accounts for (its share of the chain, measured with CUDA events on the tile stream
    # right after the timed region) divided by its launches per step.
    share = bwd[0] / chain_ms if chain_ms else None
    bwd_launches_step = nloc * max(S - 2, 0)  # this GPU's launches per step
    t_bwd_step = (ms * 1e-3) * share / bwd_launches_step if share else None
    achieved = bytes_bwd / t_bwd_step / 1e9 if t_bwd_step else None
    achieved_iso = bytes_bwd / t_bwd / 1e9 if t_bwd > 0 else None
    traffic = None
    warp_inst = None
    try:
        summ = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = summ.get("bwd_mid", {}).get("dram_bytes_per_launch")
        warp_inst = summ.get("bwd_mid", {}).get("warp_instructions")
    except Exception:
        pass
    # The pass is issue/latency bound: the same in-step launch time against the
    # instruction-issue roofline -- ncu's executed warp-instructions per launch over
    # 148 SMs x 4 schedulers x 1 warp-instruction per clock at the SM clock sampled in the run.
    issue = None
    if warp_inst and t_bwd_step:
        clk_mhz = clk.summary().get("sm_mhz") or 1965.0
        peak_issue = 148 * 4 * clk_mhz * 1e6
        issue = {"achieved_warp_inst_per_s": warp_inst / t_bwd_step, "peak": peak_issue,
                 "frac": warp_inst / t_bwd_step / peak_issue,
                 "warp_instructions_per_launch": warp_inst, "source": "profiles/ncu_summary.json"}
    flops_pass = 4 * 5 * n * np.log2(n) * n  # nominal 5 n log2 n per 1-D transform, 4 transforms per line
    # whole-path fractions (SURVEY §8(d) "Roofline fractions reported"), G GPUs:
    #   strict = probes/s x B_alg / (G x HBM), B_alg = 4N^2 (1 + 5S)  (|y|, V read fwd, V and AccBuf rmw bwd)
    #   design = probes/s x B_des / (G x HBM), B_des = 12N^2 + 36N^2 S (+ stash write/read, probe)
    #   fp32   = probes/s x 10 N^2 log2 N (4S - 2) / (G x FP32 peak), FP32 peak = SMs x 128 lanes x 2 flop
    #            x sampled SM clock (no tensor cores on this path)
    b_alg = 4 * n2 * (1 + 5 * S)
    b_des = 12 * n2 + 36 * n2 * S
    fft_flops = 10 * n2 * np.log2(n) * (4 * S - 2)
    clk_mhz = clk.summary().get("sm_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(local_rank).multi_processor_count
    fp32_peak = sms * 128 * 2 * clk_mhz * 1e6
    whole = {"strict": value * b_alg / (world * peak * 1e9), "design": value * b_des / (world * peak * 1e9),
             "fp32": value * fft_flops / (world * fp32_peak), "b_alg_bytes_per_probe": b_alg,
             "b_des_bytes_per_probe": b_des, "fft_flops_per_probe": fft_flops, "fp32_peak_tflops": fp32_peak / 1e12,
             "hbm_peak_gbs": peak}
    roofline = {"bound": "hbm", "kernel": "pass_kernel<1024, bwd_mid> (P^H, grad/AccBuf/SGD, P^H)",
                "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "algorithmic_bytes_per_launch": bytes_bwd,
                "design": {"bytes_per_launch": bytes_bwd_design,
                           "achieved": bytes_bwd_design / t_bwd_step / 1e9 if t_bwd_step else None,
                           "frac": bytes_bwd_design / t_bwd_step / 1e9 / peak if t_bwd_step else None},
                "whole_path": whole,
                "ms_per_launch_in_step": t_bwd_step * 1e3 if t_bwd_step else None,
                "share_of_chain": share, "launches_per_step": bwd_launches_step,
                "isolated": {"ms_per_launch": t_bwd * 1e3, "achieved_gbs": achieved_iso,
                             "frac": achieved_iso / peak if achieved_iso else None},
                "fwd_mid": {"ms_per_launch_isolated": t_fwd * 1e3,
                            "algorithmic_bytes_per_launch": bytes_fwd,
                            "achieved_gbs_isolated": bytes_fwd / t_fwd / 1e9 if t_fwd else None,
                            "fp32_tflops_nominal_isolated": flops_pass / t_fwd / 1e12 if t_fwd else None},
                "chain_ms_per_probe_isolated": chain_ms / 4 if chain_ms else None,
                "issue": issue}

    # ---- per-rank runtime breakdown (the paper's Fig. runtime_breakdown,
    # P:427-430): one more real iteration with serial phases, CUDA events on each rank's stream
    bd = p.profile_iteration()
    bd["rank"] = rank
    breakdown = [bd]
    if world > 1:
        allbd = [None] * world
        dist.all_gather_object(allbd, bd)
        breakdown = allbd
    # NVLink roofline of the APPP exchange (north_star: "NVLink GB/s for the halo exchange"): the
    # receivers' P2P copy kernels (bytes pulled from peer memory / their event time), against the
    # 900 GB/s nominal per direction and the pool's measured 770 GB/s peer copy (B200_PROFILING.md)
    rates = [r["nvlink_copy_gbs"] for r in breakdown if r.get("nvlink_copy_gbs")]
    nvlink = None
    if rates:
        nvlink = {"achieved_gbs": min(rates), "achieved_gbs_per_rank": rates, "peak_gbs": 900.0,
                  "peak_kind": "nominal per direction per GPU", "frac": min(rates) / 900.0,
                  "measured_peer_copy_ref_gbs": 770.0, "frac_of_measured_ref": min(rates) / 770.0,
                  "kernel": "copy2d_v4_kernel (receiver pulls the sender's AccBuf region in place)"}

    # ---- e2e: host measurements (pinned) -> device, one iteration, stitched V -> host, each step
    e2e = None
    if not args.no_e2e:
        e2e_async = args.e2e_async != "off"
        host_amp = torch.empty((nloc, n, n), dtype=torch.float32, pin_memory=True)
        p.read_measurements(0, nloc, host_amp)
        host_v = torch.empty((S, H, W), dtype=torch.float32, pin_memory=True) if rank == 0 else None
        # untimed warm-up of the e2e calls: the first stitch over ranks opens NCCL's send/recv
        # connections (0.6 s at N = 4, 0.9 s at N = 2: profiles/round2/e2e_parts.jsonl), a
        # one-time cost that is not part of a step
        p.load_measurements(host_amp, flags=PTYCHO_AMP_ASYNC if e2e_async else 0)
        p.stitch(host_v, root=0, rank=rank)
        p.synchronize()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            p.load_measurements(host_amp, flags=PTYCHO_AMP_ASYNC if e2e_async else 0)
            p.iterate()
            p.stitch(host_v, root=0, rank=rank)
        f1.record(stream)
        p.synchronize()
        barrier()
        ems = f0.elapsed_time(f1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": cfg.n_probes / (ems / 1e3), "unit": "probe-locations/s",
               "h2d_bytes_per_step": cfg.n_probes * n2 * 4, "d2h_bytes_per_step": S * H * W * 4,
               "ms_per_step": ems, "steps": args.e2e_steps, "async_upload": e2e_async}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        workers = cpu_workers()
        per = 25 if S >= 25 else S
        v, dt, sample = cpu_oracle_sample(cfg, workers, per)
        v1, dt1, sample1 = cpu_oracle_sample(cfg, 1, per)
        cpu = {"value": v, "unit": "probe-locations/s", "cores": workers, "kind": "oracle", "sample": sample,
               "seconds": dt, "cpu_model": cpu_model(), "nproc": os.cpu_count(),
               "one_thread": {"value": v1, "seconds": dt1, "sample": sample1},
               "tiny_full_iteration": cpu_tiny_iteration()}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "probe-locations/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "sec_per_iteration": ms / 1e3,
                "higher_is_better": True, "scaling": "strong",
                "vs_baseline": vs_baseline(cfg, value), "dtype": "f32", "data": "synthetic",
                "config": {"workload": workload_name(cfg),
                           "grid": f"{R}x{C}", "halo": halo, "tiles_per_gpu": ntiles // world,
                           "alpha": alpha, "pass_period": "once per iteration",
                           "l2": (f"inputs > L2 (workspace {ws / 1e9:.1f} GB per GPU vs the 126 MB L2; no flush)"
                                  if ws > 126e6 else "inputs fit in L2 (no flush): not a bench workload"),
                           "workspace_gb_per_gpu": ws / 1e9,
                           "adjoint": "stash-free (phi recomputed)" if args.stash_free else "stash",
                           "host_affinity": f"GPU-local NUMA node ({numa_cpus} CPUs)" if numa_cpus else "default"},
                "gpu_launches": launches, "roofline": roofline, "clocks": clk.summary(),
                "breakdown": {"note": "one extra iteration, APPP slab pipelining off (phases serial); ms per rank",
                              "ranks": breakdown},
                "nvlink_roofline": nvlink,
                "e2e": e2e, "cpu_baseline": cpu, "loss_after": loss, "appp": appp,
                "paper_context": "GD small LT: 2310 probe-locations/s on 462 V100 (P:65-74); "
                                 "large LT: 12600 on 4158 V100 (P:117-126)"}
        print(json.dumps(line), flush=True)
    p.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
