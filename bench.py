#!/usr/bin/env python
"""Benchmark of the fused NCM-update + FE-assembly hot path (BASELINE.json metric:
quadrature-point stress+tangent updates/s and assembled elements/s, % of the
fp64 roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl reference]

One "step" = one commet_assemble call (zeroing, every colour launch of the
fused kernel and, for N > 1, the interface exchange) over the whole mesh.
Rank 0 prints ONE JSON line.  N > 1 runs under torchrun, one rank per GPU,
z-slab partition with NCCL interface exchange (strong scaling: fixed mesh).
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

from synth import gen  # noqa: E402

METRIC = "quadrature-point stress+tangent updates/s (assembled elements/s and % fp64 roofline alongside)"
FP64_PEAK_TFLOPS = 36.9   # measured, sustained DMMA m8n8k4, profiles/r01_fp64_peak.json
FP64_PEAK_SOURCE = "measured: tools/fp64_peak.cu sustained DMMA (profiles/r01_fp64_peak.json); MEASURED_PEAKS.json has no fp64 entry"
HBM_FALLBACK_GBS = 6549.1  # only if MEASURED_PEAKS.json is absent (its value on this pool, round 2)
# DRAM bytes (read + write) per launch of the dominant kernel, from one ncu capture of the kernel
# the bench launches (profiles/r02_ncu_traffic.json: config -> kernel signature + bytes); reported
# only when the signature matches the launched kernel
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return HBM_FALLBACK_GBS, "fallback (MEASURED_PEAKS.json absent)"


def measured_traffic(config: str, kernel: str):
    """-> (bytes per launch, source) of the ncu capture of `kernel` on `config`, or (None, why)."""
    try:
        with open(TRAFFIC_FILE) as f:
            rec = json.load(f).get(config)
    except (OSError, ValueError):
        return None, "no ncu traffic record"
    if not rec:
        return None, f"no ncu traffic record for {config}"
    if rec.get("kernel") != kernel:
        return None, f"ncu record is of {rec.get('kernel')}, the bench launched {kernel}"
    return float(rec["dram_bytes_per_launch"]), rec.get("source", TRAFFIC_FILE)


def host_info():
    """CPU model, logical CPUs and RAM of the host (the cpu_baseline context)."""
    model, ram = None, None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                ram = round(int(ln.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return dict(cpu_model=model, logical_cpus=os.cpu_count(), ram_gib=ram)

WORKLOAD = {
    "c1": "c1: 4^3 hex8 unit cube, 2x2x2 Gauss (512 qp), NCM 16x2 softplus + kappa(J-1)^2, u ~ U(+-0.02)",
    "c2": "c2: 16^3 hex8 jittered 10%, 32,768 qp, NCM 32x2, smooth u amp 0.05",
    "c3": "c3: 64^3 hex8, 262,144 elements, 2,097,152 qp, 823,875 DOFs, NCM 64x3, u_x = 0.2x + smooth 0.01",
    "c4": "c4: 48^3 x 6 tet10 jittered, 663,552 elements, 2,654,208 qp, 2,738,019 DOFs, NCM 128x3, smooth u amp 0.1",
    "c5": "c5: 256^3 hex8, 16,777,216 elements, 134,217,728 qp, 50,923,779 DOFs, NCM 64x3, smooth u amp 0.05",
}


def flops_per_qp(elem_type: int, w: int, L: int) -> int:
    """NCM_min(w, L) + ELEM(n_en) (FMA = 2 flops,
    transcendentals not counted) -- the algorithmic count."""
    n_en = 8 if elem_type == gen.HEX8 else 10
    n_d = 3 * n_en
    ncm = 10 * w * w * (L - 1) + 20 * w * L + 8 * w
    elem = (18 * n_en + 100 + 350 + 54 + 18 * n_en + 54 * n_en + 72 * n_d + 14 * n_d * (n_d + 1) // 2
            + 18 * n_en + 9 * n_en * (n_en + 1) // 2)
    return ncm + elem


def hbm_bytes_per_element(elem_type: int, nnz_per_el: float, dofs_per_el: float) -> float:
    """Algorithmic HBM bytes per element (write-once outputs): dN/dX + w + conn
    + slots + u gather + r + CSR values."""
    n_en, n_q = (8, 8) if elem_type == gen.HEX8 else (10, 4)
    return 8 * n_q * n_en * 3 + 8 * n_q + 4 * n_en + n_en * n_en + 8 * dofs_per_el + 8 * nnz_per_el + \
        8 * dofs_per_el


# ---------------------------------------------------------------------------
# distributed helpers
# ---------------------------------------------------------------------------
def gpu_local_cpus(device: int):
    """CPUs of the GPU's NUMA node (sysfs local_cpulist of its PCI function), or None if unknown."""
    try:
        import pynvml
        pynvml.nvmlInit()
        bus = pynvml.nvmlDeviceGetPciInfo(pynvml.nvmlDeviceGetHandleByIndex(device)).busId
        bus = (bus.decode() if isinstance(bus, bytes) else bus).lower()
        cpus = set()
        with open(f"/sys/bus/pci/devices/{bus[-12:]}/local_cpulist") as f:
            for part in f.read().strip().split(","):
                a, _, b = part.partition("-")
                cpus.update(range(int(a), int(b or a) + 1))
        return cpus & os.sched_getaffinity(0) or None
    except Exception:
        return None


class numa_local:
    """Allocate pinned host buffers from the GPU's NUMA node: the pages of a cudaHostAlloc are placed
    by the allocating thread (first touch), and a remote node puts the inter-socket link in front of
    every host<->device copy.  Restores the process's CPU affinity on exit."""

    def __init__(self, device: int):
        self.cpus = gpu_local_cpus(device)

    def __enter__(self):
        self.saved = os.sched_getaffinity(0)
        if self.cpus:
            os.sched_setaffinity(0, self.cpus)
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.saved)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def launch_plan(gpus: int, env: dict, device_count: int, needs_gpus: bool = True):
    """What `bench.py --gpus N` does in this process: ("run", None) -- this process is one
    of the N ranks (or N = 1); ("relaunch", None) -- re-run itself under torch.distributed.run
    with N ranks (WORLD_SIZE unset, N > 1); ("refuse", why) -- --gpus disagrees with the
    launcher's WORLD_SIZE, or fewer than N devices are visible (a silent 1-GPU line labelled
    N GPUs would be wrong)."""
    if gpus < 1:
        return "refuse", f"--gpus {gpus} < 1"
    ws = env.get("WORLD_SIZE")
    if ws is not None and int(ws) != gpus:
        return "refuse", f"--gpus {gpus} but the launcher started WORLD_SIZE={ws} ranks"
    if needs_gpus and device_count < gpus:
        return "refuse", f"--gpus {gpus} but only {device_count} CUDA device(s) are visible"
    if ws is None and gpus > 1:
        return ("relaunch", None) if needs_gpus else ("run", None)
    return "run", None


def relaunch_cmd(gpus: int, argv: list, port: int):
    """torch.distributed.run command line that re-runs this script with `gpus` ranks on this node."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        self.p = None
        self.index = index
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle as it stands, on a bounded sample
# ---------------------------------------------------------------------------
def oracle_sample(cfg: dict, seconds: float):
    """Time oracle.assemble (OpenMP over colours, all host cores) on the first
    n_s elements of the workload, n_s sized for ~`seconds` of CPU work."""
    import oracle
    conn, gN, qw = cfg["conn"], cfg["gradN"], cfg["qp_w"]
    n_q = gN.shape[1]

    def run(ns):
        sub = np.ascontiguousarray(conn[:ns])
        rp, ci = oracle.pattern(cfg["n_nodes"], sub)
        t0 = time.perf_counter()
        oracle.assemble(cfg["ncm"], cfg["n_nodes"], sub, gN[:ns], qw[:ns], cfg["u"], rp, ci, mode=1)
        return time.perf_counter() - t0

    ns = min(conn.shape[0], 256)
    t = run(ns)
    while t < 0.5 and ns < conn.shape[0]:
        ns = min(conn.shape[0], ns * 4)
        t = run(ns)
    ns2 = int(min(conn.shape[0], max(ns, ns * seconds / max(t, 1e-9))))
    if ns2 != ns:
        ns, t = ns2, run(ns2)
    cores = oracle.max_threads()
    # per-core rate: one thread on a sample of ~2 s (then the thread count is restored)
    ns1 = int(max(16, min(ns, ns * 2.0 / max(t * cores, 1e-9))))
    sub1 = np.ascontiguousarray(conn[:ns1])
    rp1, ci1 = oracle.pattern(cfg["n_nodes"], sub1)
    t1 = time.perf_counter()
    oracle.assemble(cfg["ncm"], cfg["n_nodes"], sub1, gN[:ns1], qw[:ns1], cfg["u"], rp1, ci1, mode=1, n_threads=1)
    t1 = time.perf_counter() - t1
    oracle.assemble(cfg["ncm"], cfg["n_nodes"], sub1[:1], gN[:1], qw[:1], cfg["u"], *oracle.pattern(cfg["n_nodes"], sub1[:1]),
                    mode=1, n_threads=cores)
    host = dict(host_info(), single_thread_qp_s=ns1 * n_q / t1,
                single_thread_sample=f"first {ns1} elements, 1 thread, {t1:.2f} s")
    return dict(value=ns * n_q / t, unit="qp/s", cores=cores, kind="oracle",
                sample=f"first {ns} of {conn.shape[0]} elements ({ns * n_q} qp), oracle.assemble "
                       f"(plain C, OpenMP over element colours), {t:.1f} s",
                host=host, elements_per_s=ns / t, seconds=t)


def run_reference(args):
    """--impl reference: the oracle as it stands, timed on the host cores on a
    bounded sample of the same workload each step (rank 0 only)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = gen.make_config(args.config)
    per_step = max(2.0, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    base = oracle_sample(cfg, per_step)                 # sizes the sample
    ns = int(base["sample"].split()[1])
    import oracle
    sub = np.ascontiguousarray(cfg["conn"][:ns])
    rp, ci = oracle.pattern(cfg["n_nodes"], sub)
    n_q = cfg["gradN"].shape[1]
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.assemble(cfg["ncm"], cfg["n_nodes"], sub, cfg["gradN"][:ns], cfg["qp_w"][:ns], cfg["u"],
                        rp, ci, mode=1)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    value = ns * n_q / t
    line = dict(impl="reference", metric=METRIC, value=value, unit="qp/s", n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, ms_per_step=t * 1e3, higher_is_better=True, scaling="strong",
                vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=WORKLOAD[args.config], sample_elements=ns),
                elements_per_s=ns / t,
                cpu_baseline=dict(value=value, unit="qp/s", cores=oracle.max_threads(), kind="oracle",
                                  sample=f"first {ns} elements of {args.config} per step", host=base["host"]),
                e2e=dict(value=value, unit="qp/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# the GPU path
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(WORKLOAD))
    ap.add_argument("--impl", default="commet", choices=["commet", "reference"])
    ap.add_argument("--kernel", default="fused", choices=["fused", "simple"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--jitter", type=float, default=None,
                    help="override the config's node jitter (fraction of h): every element then has its own dN/dX")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="N > 1: interface rows over NCCL send/recv + unpack (default), or added straight "
                         "into the owner's buffers by the kernels over NVLink P2P (CUDA IPC)")
    args = ap.parse_args()
    ndev = 0
    if args.impl != "reference" or "WORLD_SIZE" in os.environ:
        import torch
        ndev = torch.cuda.device_count() if args.impl != "reference" else 0
    action, why = launch_plan(args.gpus, dict(os.environ), ndev, needs_gpus=args.impl != "reference")
    if action == "refuse":
        print(f"bench.py: {why}", file=sys.stderr, flush=True)
        return 2
    if action == "relaunch":
        return subprocess.call(relaunch_cmd(args.gpus, sys.argv[1:], _free_port()))
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2510_00884_b200 as pc

    spec = gen.CONFIGS[args.config]
    comm = None
    if ws > 1:
        cfg = gen.slab_partition(args.config, ws, rank)   # z-slab r of ws, with ghost layer
        comm = pc.nccl_comm_from_process_group(rank, ws, local)
    else:
        cfg = gen.make_config(args.config, jitter=args.jitter)
    lib = pc.Commet(cfg, cfg["ncm"], device=local, nccl_comm=comm)
    if args.kernel == "simple":
        lib.set_kernel(pc.KERNEL_SIMPLE)
    n_el, n_q = cfg["conn"].shape[0], cfg["gradN"].shape[1]
    info = lib.info()
    kinfo = lib.kernel_info()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    with numa_local(local) as nl:
        u_host = torch.from_numpy(cfg["u"]).pin_memory()
    u = u_host.to(dev)
    r, v = lib.alloc_outputs()
    peer = ws > 1 and args.exchange == "peer"
    if peer:  # the kernels add halo rows into the owners' (r, v) over NVLink; barriers inside assemble
        pc.setup_peer_exchange(lib, r, v, rank, ws)
    lib.set_timing(args.steps)

    # warm-up + correctness gate (det F > 0 everywhere)
    for _ in range(args.warmup):
        lib.assemble(u, r, v)
    torch.cuda.synchronize()
    bad = lib.check()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # ---- timed region: K device-resident steps --------------------------------------------
    clk = Clocks(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        lib.assemble(u, r, v)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / args.steps
    kern_ms = float(np.mean(lib.kernel_times(args.steps)))
    t_local = torch.tensor([ms, kern_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms, kern_ms = float(t_local[0]), float(t_local[1])

    # ---- e2e: host u -> device, assemble, device -> host r and CSR values ----------------------
    # every step copies u H2D (pinned) and reads r and the CSR values back D2H (pinned); two
    # device output sets and a copy stream let step s's D2H overlap step s+1's assembly
    e2e = None
    if not args.no_e2e and not peer:
        # the library's host-buffer call (commet_assemble_host): it uploads u, assembles and reads
        # r and the CSR values back, overlapping call s's read-back and call s+1's upload with
        # call s+1's assembly over its own two device staging sets (so the bench's set goes first)
        n_rows, nnz = r.numel(), v.numel()
        del r, v
        torch.cuda.empty_cache()
        with numa_local(local):
            r_host = torch.empty(n_rows, dtype=torch.float64).pin_memory()
            v_host = torch.empty(nnz, dtype=torch.float64).pin_memory()
        lib.assemble_host(u_host, r_host, v_host, stream)  # allocates the staging sets (untimed)
        lib.host_wait()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            lib.assemble_host(u_host, r_host, v_host, stream)
        lib.host_wait(stream)
        f1.record(stream)
        torch.cuda.synchronize()
        ms_e2e = f0.elapsed_time(f1) / args.steps
        t_e = torch.tensor([ms_e2e], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        ms_e2e = float(t_e[0])
        e2e = dict(value=spec_total_qp(args.config, n_el, n_q, ws) / (ms_e2e * 1e-3), unit="qp/s",
                   h2d_bytes_per_step=u_host.numel() * 8, d2h_bytes_per_step=(n_rows + nnz) * 8,
                   ms_per_step=ms_e2e,
                   host_buffers_cpus=(f"GPU-local NUMA node, {len(nl.cpus)} CPUs" if nl.cpus else "affinity unchanged"),
                   note="commet_assemble_host on pinned host buffers (C ABI): per call the library uploads "
                        "u, assembles and reads r + CSR values back; two device staging sets overlap call "
                        "s's read-back and call s+1's upload with call s+1's assembly")
        del r_host, v_host
    elif not args.no_e2e:  # peer mode: the peers hold this rank's registered (r, v)
        with numa_local(local):
            r_host = torch.empty(r.numel(), dtype=torch.float64).pin_memory()
            v_host = torch.empty(v.numel(), dtype=torch.float64).pin_memory()
        # peer mode: the peers hold this rank's registered (r, v), so one output set (the
        # read-back of step s finishes before step s+1 assembles)
        sets = [(r, v), (r, v) if peer else lib.alloc_outputs()]
        # the read-back is split over NCS copy streams (chunks of the CSR values round-robin):
        # one cudaMemcpyAsync uses one copy engine, several keep the host link busier
        NCS = int(os.environ.get("COMMET_E2E_STREAMS", "2"))
        copy_streams = [torch.cuda.Stream(dev) for _ in range(NCS)]
        done_c = [torch.cuda.Event(), torch.cuda.Event()]
        # the H2D of step s's u runs on its own stream into one of two device copies, so it
        # overlaps the assembly of step s-1 (the copy of step s waits for step s-2's assembly)
        u_sets = [u, torch.empty_like(u)]
        h2d = torch.cuda.Stream(dev)
        done_h = [torch.cuda.Event(), torch.cuda.Event()]
        done_d = [[torch.cuda.Event() for _ in range(NCS)] for _ in range(2)]
        nchunk = 4 * NCS
        vchunks = [(i * v.numel() // nchunk, (i + 1) * v.numel() // nchunk) for i in range(nchunk)]
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for s_ in range(args.steps):
            k = s_ % 2
            if s_ >= 2:
                for ev in done_d[k]:
                    stream.wait_event(ev)
            if peer and s_ >= 1:  # single output set: the previous read-back must be done
                for ev in done_d[1 - k]:
                    stream.wait_event(ev)
            if s_ >= 2:
                h2d.wait_event(done_c[k])
            with torch.cuda.stream(h2d):
                u_sets[k].copy_(u_host, non_blocking=True)
            done_h[k].record(h2d)
            stream.wait_event(done_h[k])
            lib.assemble(u_sets[k], *sets[k])
            done_c[k].record(stream)
            for cs in copy_streams:
                cs.wait_event(done_c[k])
            with torch.cuda.stream(copy_streams[0]):
                r_host.copy_(sets[k][0], non_blocking=True)
            for ci, (a0, a1) in enumerate(vchunks):
                with torch.cuda.stream(copy_streams[ci % NCS]):
                    v_host[a0:a1].copy_(sets[k][1][a0:a1], non_blocking=True)
            for ci, cs in enumerate(copy_streams):
                done_d[k][ci].record(cs)
        for cs in copy_streams:
            stream.wait_stream(cs)
        f1.record(stream)
        torch.cuda.synchronize()
        ms_e2e = f0.elapsed_time(f1) / args.steps
        t_e = torch.tensor([ms_e2e], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        ms_e2e = float(t_e[0])
        e2e = dict(value=spec_total_qp(args.config, n_el, n_q, ws) / (ms_e2e * 1e-3), unit="qp/s",
                   h2d_bytes_per_step=u_host.numel() * 8, d2h_bytes_per_step=(r.numel() + v.numel()) * 8,
                   ms_per_step=ms_e2e,
                   note=f"pinned host buffers; H2D of step s+1 and D2H of step s overlap the assembly "
                        f"of step s+1 (two device input and output sets, 1 + {NCS} copy streams)")
        del sets, u_sets

    total_qp = spec_total_qp(args.config, n_el, n_q, ws)
    total_el = total_qp // n_q
    fl = flops_per_qp(cfg["elem_type"], spec.width, spec.n_hidden)
    # roofline of the dominant kernel (all its colour launches of one step; the launches are equal
    # in size, so the per-launch rate is the per-step rate)
    achieved = fl * total_qp / ws / (kern_ms * 1e-3) / 1e12
    kname = ("ws_kernel" if kinfo.get("warp_specialised") else "fused_kernel") + \
        f"<w={spec.width},L={spec.n_hidden},{'hex8' if cfg['elem_type'] == gen.HEX8 else 'tet10'}," \
        f"q={kinfo.get('qps_network_batch')}/{kinfo.get('qps_element_batch')}>"
    traffic, traffic_src = measured_traffic(args.config, kname) if ws == 1 and args.kernel == "fused" else \
        (None, "single-GPU fused kernel only")
    hbm_pk, hbm_src = hbm_peak()
    nnz_local, rows_local = lib.nnz, lib.n_rows
    hbm = hbm_bytes_per_element(cfg["elem_type"], nnz_local / max(n_el, 1), rows_local / max(n_el, 1))
    line = dict(
        metric=METRIC, value=total_qp / (ms * 1e-3), unit="qp/s", n_gpus=ws, steps=args.steps,
        warmup=args.warmup, ms_per_step=ms, higher_is_better=True, scaling="strong", vs_baseline=None,
        dtype="f64", data="synthetic (seeded mesh, NCM weights N(0,0.3^2), displacement; synth/gen.py)",
        config=dict(workload=WORKLOAD[args.config] + (f", nodes jittered {args.jitter:g} h" if args.jitter else ""),
                    elements=total_el, qp=total_qp, nnz_rank0=nnz_local,
                    width=spec.width, hidden_layers=spec.n_hidden, colours=info["n_colours"],
                    kernel=args.kernel, launch=kinfo,
                    parallelism=(f"z-slabs x{ws}, interface rows over " + ("NVLink P2P (peer mode)" if peer else "NCCL"))
                    if ws > 1 else "single GPU",
                    l2="inputs larger than L2 (dN/dX + CSR values >> 126 MB), no flush needed"
                    if args.config in ("c3", "c4", "c5") else "inputs fit in L2 (latency-bound config)"),
        elements_per_s=total_el / (ms * 1e-3),
        kernel_ms_per_step=kern_ms,
        roofline=dict(bound="alu", pipe="fp64 (DFMA/DMMA share one datapath)", achieved=achieved,
                      peak=FP64_PEAK_TFLOPS, unit="TFLOP/s", frac=achieved / FP64_PEAK_TFLOPS,
                      traffic=traffic, traffic_unit="bytes per launch (one colour launch of " + kname +
                      "; ncu dram__bytes_read.sum + dram__bytes_write.sum)", traffic_source=traffic_src,
                      algorithmic_bytes_per_launch=hbm * n_el / max(info["n_colours"], 1),
                      kernel=kname, flops_per_qp=fl, peak_source=FP64_PEAK_SOURCE,
                      hbm_algorithmic_gbs=hbm * n_el / (kern_ms * 1e-3) / 1e9, hbm_peak_gbs=hbm_pk,
                      hbm_peak_source=hbm_src),
        clocks=clocks, gpu_launches=info["launches"] * args.steps,
        e2e=e2e, det_f_ok=(bad == -1),
    )
    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = {k: v for k, v in oracle_sample(cfg, args.cpu_seconds).items()
                                if k in ("value", "unit", "cores", "kind", "sample", "host")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        lib.close()
        pc.nccl_comm_destroy(comm)
        dist.destroy_process_group()
    return 0


def spec_total_qp(name, n_el_local, n_q, ws):
    spec = gen.CONFIGS[name]
    if ws == 1:
        return n_el_local * n_q
    per_cell = 1 if spec.elem_type == gen.HEX8 else 6
    return spec.n ** 3 * per_cell * n_q


if __name__ == "__main__":
    sys.exit(main())
