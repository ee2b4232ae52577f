#!/usr/bin/env python
"""Headline benchmark: radius-search queries/sec on the BASELINE config-1
cloud (20M-point ALS tile + 200 buildings, cell 1 m), sphere r = 1 m, every
point a query, full sorted CSR neighbour lists; plus index build ms.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One JSON line on rank 0:
  value  : queries/sec over all ranks, inputs resident in HBM, device time
           (CUDA events on the launching stream, max over ranks)
  e2e    : the same metric through the C ABI with HOST buffers: pinned
           query coordinates in, full CSR (row_ptr + cols) back to pinned
           host memory, both copies inside the timed region
  roofline: dominant kernel's algorithmic bytes (24 B x the reference's
           points_tested) / its event-timed duration, against
           MEASURED_PEAKS.json hbm_gbs
  cpu_baseline: the reference library compiled from its own sources
           (oracle/_ref) on this host's cores, on a bounded query sample

Multi-GPU (torchrun): replicated index, queries sharded in contiguous blocks
(strong scaling; no data-path collective). --impl reference: rank 0 times the
reference's own CPU implementation, other ranks exit.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLAVORS = {"dense": 0, "sparse": 1, "mixed": 2}
KERNELS = {"sphere": 0, "cube": 1}
FALLBACK_HBM_GBS = 6650.0
BAD_REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--scale", type=float, default=1.0, help="shrink the cloud (tests only)")
    ap.add_argument("--radius", type=float, default=1.0)
    ap.add_argument("--kernel", default="sphere", choices=list(KERNELS))
    ap.add_argument("--flavor", default="mixed", choices=list(FLAVORS))
    ap.add_argument("--cpu-sample", type=int, default=1_000_000,
                    help="queries per CPU-baseline / reference step")
    ap.add_argument("--layout", default="replicated", choices=["replicated", "slabs"],
                    help="slabs: x-slab partition with halo exchange through cm_build_slab "
                         "(config 4's layout)")
    ap.add_argument("--halo", type=float, default=5.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def workload_name(a):
    return (f"cfg{a.config} ALS {int(20_000_000 * a.scale)} pts +buildings, cell 1 m, "
            f"{a.kernel} r={a.radius:g} m, every point a query, sorted CSR")


def read_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_lib():
    """The reference compiled from its own sources if present, else the port."""
    from oracle.oracle import lib
    try:
        return lib("reference"), "reference"
    except FileNotFoundError:
        return lib("oracle"), "port"


def run_cpu(cloud, a, steps, warmup, threads=0, flavor=None):
    """Times the CPU implementation on bounded query samples. Returns a dict."""
    from oracle.oracle import CpuIndex
    L, kind = cpu_reference_lib()
    flavor = flavor or a.flavor
    t0 = time.perf_counter()
    idx = CpuIndex(cloud, flavor=FLAVORS[flavor], which=kind)
    build_s = time.perf_counter() - t0
    nthreads = threads or os.cpu_count() or 1
    stride = max(1, cloud.shape[0] // a.cpu_sample)
    rates = []
    for s in range(warmup + steps):
        q = np.ascontiguousarray(cloud[(s % stride)::stride][: a.cpu_sample])
        t0 = time.perf_counter()
        idx.radius(q, KERNELS[a.kernel], a.radius, threads=nthreads)
        dt = time.perf_counter() - t0
        if s >= warmup:
            rates.append(q.shape[0] / dt)
    return dict(value=statistics.median(rates), kind=kind, cores=nthreads, build_ms=build_s * 1e3,
                sample=f"{min(a.cpu_sample, cloud.shape[0])} of the {cloud.shape[0]} queries "
                       f"(every {stride}th point, a different offset per step), {flavor} map, "
                       f"{nthreads} threads, median of {steps} steps after {warmup} warm-up; "
                       f"build single-threaded")


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2502_11602_b200 import synth
    cloud = synth.config_cloud(a.config, a.scale)
    r = run_cpu(cloud, a, a.steps, a.warmup)
    line = {
        "impl": "reference", "metric": "radius-search queries/sec (20M-pt ALS, r=1 m)",
        "value": r["value"], "unit": "queries/s", "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded config-1 generator)",
        "config": {"workload": workload_name(a), "flavor": a.flavor, "n_points": int(cloud.shape[0])},
        "build_ms": {a.flavor: r["build_ms"]},
        "cpu_baseline": {"value": r["value"], "unit": "queries/s", "cores": r["cores"],
                         "kind": r["kind"], "sample": r["sample"]},
        "e2e": {"value": r["value"], "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)


def slab_arm(a):
    """x-slabs: every rank passes a contiguous 1/N
    block of the cloud (global ids = handles) to cm_build_slab, which
    all-reduces the global box, exchanges points into x-slabs + halos over
    NCCL and indexes them on the global grid; each rank then answers every
    point it owns (cm_slab_radius_search, q = NULL). value = all points /
    max-over-ranks device time; build_ms = max over ranks of device-resident
    points -> ready slab index, exchange included."""
    import torch
    import torch.distributed as dist

    from paper_2502_11602_b200 import synth
    from paper_2502_11602_b200 import cheesemap as cm
    from paper_2502_11602_b200.cluster import Cluster, Slab

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    total_mem = torch.cuda.get_device_properties(local).total_memory
    cm.pool_configure(local, int(total_mem * 0.75), min(32 << 30, int(total_mem * 0.2)))
    uid = [Cluster.unique_id("nccl") if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    cl = Cluster(uid[0], world, rank, local, "nccl")
    cloud = synth.config_cloud(a.config, a.scale)
    n = cloud.shape[0]
    lo, hi = n * rank // world, n * (rank + 1) // world
    share = torch.from_numpy(np.ascontiguousarray(cloud[lo:hi])).to(dev)
    del cloud
    stream = torch.cuda.current_stream(dev)
    kernel = KERNELS[a.kernel]
    opts = cm.BuildOptions(flavor=cm.Flavor(FLAVORS[a.flavor]))

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def allred(x, op):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    builds = []
    slab = None
    for _ in range(3):
        barrier()
        slab = None
        slab = Slab(cl, share, gid_base=lo, opts=opts, halo=a.halo, stream=stream)
        builds.append(slab.info()["timing"]["total_ms"])
    inf = slab.info()
    build_ms = allred(min(builds), dist.ReduceOp.MAX if world > 1 else None)
    n_owned = inf["n_owned"]
    L = cm._native.lib()
    import ctypes

    def step():
        csr = ctypes.c_void_p()
        cm._check(L.cm_slab_radius_search(slab._h, None, n_owned, kernel, a.radius,
                                          ctypes.c_void_p(stream.cuda_stream), ctypes.byref(csr)))
        return csr

    for _ in range(a.warmup):
        L.cm_csr_free(step())
    nnz = ctypes.c_uint64()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize(dev)
    launches0 = cm._native.launch_count()
    ms = []
    for _ in range(a.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        csr = step()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
        L.cm_csr_info(csr, None, ctypes.byref(nnz), None, None)
        L.cm_csr_free(csr)
    launches = (cm._native.launch_count() - launches0) // a.steps
    barrier()
    clk = clocks.stop()
    t = allred(sum(ms) / len(ms), dist.ReduceOp.MAX if world > 1 else None)
    nnz_all = allred(float(nnz.value), dist.ReduceOp.SUM if world > 1 else None)
    halo_all = allred(float(inf["n_halo"]), dist.ReduceOp.SUM if world > 1 else None)
    if rank == 0:
        emit({
            "metric": f"radius-search queries/sec (cfg{a.config} x-slabs, r={a.radius:g} m)",
            "value": round(n / (t * 1e-3), 1), "unit": "queries/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(t, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (seeded config-{a.config} generator, DESIGN.md)",
            "config": {"workload": f"cfg{a.config} ALS {n} pts, x-slabs x{world}, halo "
                                   f"{a.halo:g} m, {a.kernel} r={a.radius:g} m, every point a "
                                   "query (its owner rank), sorted CSR in global ids",
                       "flavor": a.flavor, "layout": "slabs", "n_points": n,
                       "neighbours": int(nnz_all), "halo_points": int(halo_all),
                       "l2": "flushed (256 MB write) before every timed step",
                       "call": "cm_build_slab + cm_slab_radius_search (q = NULL: owned points)"},
            "build_ms": round(build_ms, 3),
            "build_note": "max over ranks: device-resident share -> ready slab index, bbox "
                          "all-reduce + point exchange included (host->device share copy "
                          "excluded)",
            "gpu_launches": int(launches), "clocks": clk})
    del slab
    if world > 1:
        dist.destroy_process_group()


_JSON_OUT = None


def emit(line):
    """The bench line, to the process's original stdout."""
    print(json.dumps(line), file=_JSON_OUT or sys.stdout, flush=True)


def main():
    # stdout carries exactly one JSON line: everything else written to file
    # descriptor 1 (NCCL prints its version banner there when NCCL_DEBUG is
    # set, as on the GPU boxes) goes to stderr
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    a = parse()
    if a.impl == "reference":
        reference_arm(a)
        return
    if a.layout == "slabs":
        slab_arm(a)
        return
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2502_11602_b200 import _native, synth
    from paper_2502_11602_b200 import cheesemap as cm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; BENCH_DIST_BACKEND=gloo lets several ranks share
    # one GPU for a functional check of the N > 1 path (no kernel waits on
    # another rank: collectives run on the host)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev if backend == "nccl" else torch.device("cpu")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    L = _native.lib()
    # This process owns the GPU: let the library's private pool keep 3/4 of
    # HBM cached and reserve 32 GiB up front (cm_pool_configure; the library
    # default keeps 1/8 and reserves nothing)
    total_mem = torch.cuda.get_device_properties(local).total_memory
    pool_keep, pool_reserve = int(total_mem * 0.75), min(32 << 30, int(total_mem * 0.2))
    cm.pool_configure(local, pool_keep, pool_reserve)
    t0 = time.perf_counter()
    cloud = synth.config_cloud(a.config, a.scale)
    log(f"[rank {rank}] generated {cloud.shape[0]} points in {time.perf_counter() - t0:.1f}s")
    d_cloud = torch.from_numpy(cloud).to(dev)
    stream = torch.cuda.current_stream(dev)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    kernel = KERNELS[a.kernel]

    # ---- index build (device-resident points -> ready index), per flavour
    build_ms = {}
    build_detail = {}
    index = None
    for name in ("sparse", "mixed", "dense"):
        best = None
        for _ in range(3):
            m = cm.Cheesemap.build(d_cloud, cm.BuildOptions(flavor=cm.Flavor(FLAVORS[name])),
                                   device=local, stream=stream)
            t = m.build_timing()
            if best is None or t["total_ms"] < best["total_ms"]:
                best = t
            if name == a.flavor:
                index = m
            else:
                del m
        build_ms[name] = allmax(best["total_ms"])
        build_detail[name] = {k: round(v, 3) for k, v in best.items()}
    log(f"[rank {rank}] build ms {build_ms}")
    # SURVEY 8d build bytes: 24N read + 24N + 4N written (sorted xyz + u32
    # ids) + the flavour's table (dense 8(V+1), sparse / mixed 16U); reported,
    # the >= 50 % target is for the query kernels
    occ = index.occupancy_stats()
    n_pts = int(cloud.shape[0])
    peak_b, _ = read_peak()
    build_roof = {}
    for name, ms_b in build_ms.items():
        tb = 8 * (int(occ["total_voxels"]) + 1) if name == "dense" else 16 * int(occ["non_empty"])
        bb = 52 * n_pts + tb
        build_roof[name] = {"alg_bytes": bb, "achieved_gbs": round(bb / (ms_b * 1e-3) / 1e9, 1),
                            "frac": round(bb / (ms_b * 1e-3) / 1e9 / peak_b, 4)}

    # ---- this rank's queries: an equal-count x-slab of the cloud, so each
    # rank's share stays spatially dense (query tiles stay compact)
    nq_total = cloud.shape[0]
    lo = nq_total * rank // world
    hi = nq_total * (rank + 1) // world
    if world > 1:
        shard = torch.argsort(d_cloud[:, 0], stable=True)[lo:hi]
        q_dev = d_cloud[shard].contiguous()
        shard_host = shard.cpu().numpy()
    else:
        # centres in a buffer of their own: the general path (key sort of the
        # centres); the headline at N = 1 is cm_radius_search_self
        q_dev = d_cloud.clone()
        shard_host = None
    nq = hi - lo
    self_q = world == 1

    # algorithmic bytes: 24 B x the reference's points_tested for these queries
    tested = torch.zeros(nq, dtype=torch.int64, device=dev)
    counts = torch.zeros(nq, dtype=torch.int32, device=dev)
    cm._check(L.cm_radius_count(index.handle, ctypes.c_void_p(q_dev.data_ptr()), nq, kernel,
                                a.radius, ctypes.c_void_p(counts.data_ptr()),
                                ctypes.c_void_p(tested.data_ptr()), sptr))
    torch.cuda.synchronize(dev)
    sum_tested = int(tested.sum().item())
    nnz_rank = int(counts.to(torch.int64).sum().item())
    alg_bytes = 24 * sum_tested
    del tested, counts

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step_general():
        csr = ctypes.c_void_p()
        cm._check(L.cm_radius_search(index.handle, ctypes.c_void_p(q_dev.data_ptr()), nq, kernel,
                                     a.radius, sptr, ctypes.byref(csr)))
        return csr

    def step_self():
        csr = ctypes.c_void_p()
        cm._check(L.cm_radius_search_self(index.handle, kernel, a.radius, sptr, ctypes.byref(csr)))
        return csr

    step_device = step_self if self_q else step_general

    for _ in range(a.warmup):
        csr = step_device()
        torch.cuda.synchronize(dev)
        L.cm_csr_free(csr)
    _native.query_stats(reset=True)
    csr = step_device()
    torch.cuda.synchronize(dev)
    L.cm_csr_free(csr)
    step_stats = _native.query_stats(reset=True)  # one step: count + fill passes

    # ---- timed region (device-resident inputs)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize(dev)
    launches0 = _native.launch_count()
    step_ms, kern = [], []
    for _ in range(a.steps):
        flush.zero_()  # L2 flush (256 MB write) outside the timed events
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        csr = step_device()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        kern.append(_native.last_query_timing())
        L.cm_csr_free(csr)
    torch.cuda.synchronize(dev)
    launches = (_native.launch_count() - launches0) // a.steps
    barrier()
    clk = clocks.stop()
    ms_rank = sum(step_ms) / len(step_ms)
    ms = allmax(ms_rank)
    value = nq_total / (ms * 1e-3)

    # the same workload with the centres in a caller buffer (the general
    # path: centre-key sort + the same kernels), reported beside the headline
    general = None
    if self_q:
        for _ in range(2):
            L.cm_csr_free(step_general())
        g_ms = []
        for _ in range(a.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            csr = step_general()
            e1.record(stream)
            e1.synchronize()
            g_ms.append(e0.elapsed_time(e1))
            L.cm_csr_free(csr)
        gm = sum(g_ms) / len(g_ms)
        general = {"value": round(nq_total / (gm * 1e-3), 1), "unit": "queries/s",
                   "ms_per_step": round(gm, 4),
                   "call": "cm_radius_search with the centres in a separate device buffer "
                           "(cell-key radix sort of the centres inside the step)"}

    def mean_of(key):
        return sum(k[key] for k in kern) / len(kern)

    phase = {k: round(mean_of(k), 4) for k in ("order_ms", "pass1_ms", "rowsort_ms", "scan_ms",
                                                "pass2_ms")}
    two_pass = any(k["two_pass"] == 1 for k in kern)
    phase["two_pass"] = bool(two_pass)
    dom = "pass1_ms"
    dom_ms = phase[dom]
    peak, peak_src = read_peak()
    achieved = alg_bytes / (dom_ms * 1e-3) / 1e9
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            traffic = tj.get(f"{a.flavor}/collect/r{a.radius:g}")
            traffic_src = ("not measured in this run: ncu dram__bytes_read.sum + "
                           "dram__bytes_write.sum of this kernel from " +
                           tj.get("_source", "profiles/traffic.json"))
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_source": traffic_src,
                "kernel": "radius_tile_kernel<" + a.flavor + ", " +
                          ("COUNT (two-pass fallback)" if two_pass else "COLLECT") + ">",
                "kernel_ms": dom_ms, "alg_bytes_per_launch": alg_bytes,
                "peak_source": peak_src,
                "basis": "24 B x sum of the reference's points_tested (search.hpp:116) "
                         "over this launch's queries"}

    # ---- end to end through the C ABI with host buffers
    e2e = None
    if not a.no_e2e:
        q_host = torch.from_numpy(np.ascontiguousarray(
            cloud if shard_host is None else cloud[shard_host])).pin_memory()
        row_host = torch.empty(nq + 1, dtype=torch.int64).pin_memory()
        cols_host = torch.empty(max(nnz_rank, 1), dtype=torch.int32).pin_memory()

        nnz_host = ctypes.c_uint64()

        def step_e2e():
            cm._check(L.cm_radius_search_to_host(
                index.handle, ctypes.c_void_p(q_host.data_ptr()), nq, kernel, a.radius,
                ctypes.c_void_p(row_host.data_ptr()), ctypes.c_void_p(cols_host.data_ptr()),
                cols_host.numel(), ctypes.byref(nnz_host), sptr))

        for _ in range(max(1, a.warmup)):
            step_e2e()
        barrier()
        torch.cuda.synchronize(dev)
        e2e_ms = []
        for _ in range(a.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step_e2e()
            e1.record(stream)
            e1.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
        barrier()
        # median over the timed steps (one step can catch host-side noise:
        # pinned-page or PCIe contention left by the previous process)
        e2e_t = allmax(statistics.median(e2e_ms))
        e2e = {"value": nq_total / (e2e_t * 1e-3), "unit": "queries/s",
               "h2d_bytes_per_step": int(allsum(nq * 24)),
               "d2h_bytes_per_step": int(allsum((nq + 1) * 8 + nnz_rank * 4)),
               "ms_per_step": round(e2e_t, 3), "ms_steps": [round(x, 2) for x in e2e_ms],
               "statistic": "median of the timed steps, max over ranks",
               "call": "cm_radius_search_to_host (pinned host queries in, sorted CSR to pinned "
                       "host memory, chunked copy/compute overlap)"}

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        try:
            r = run_cpu(cloud, a, steps=3, warmup=1)
            cpu = {"value": r["value"], "unit": "queries/s", "cores": r["cores"],
                   "kind": r["kind"], "sample": r["sample"],
                   "build_ms": {a.flavor: round(r["build_ms"], 1)}}
            if a.flavor != "dense":  # the CPU's fastest flavour, for context
                rd = run_cpu(cloud, a, steps=3, warmup=1, flavor="dense")
                cpu["dense_map"] = {"value": rd["value"], "sample": rd["sample"],
                                    "build_ms": round(rd["build_ms"], 1)}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "queries/s", "cores": None, "kind": None,
                   "sample": f"unavailable: {ex}"}

    nnz_total = int(allsum(nnz_rank))
    if rank == 0:
        line = {
            "metric": "radius-search queries/sec (20M-pt ALS, r=1 m)",
            "value": round(value, 1), "unit": "queries/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded config-1 generator, DESIGN.md)",
            "config": {"workload": workload_name(a), "flavor": a.flavor,
                       "n_points": int(cloud.shape[0]), "n_queries": nq_total,
                       "neighbours": nnz_total, "radius_m": a.radius, "kernel": a.kernel,
                       "l2": "flushed (256 MB write) before every timed step",
                       "parallelism": f"replicated index, queries sharded x{world} "
                                      "(equal-count x-slabs)",
                       "call": ("cm_radius_search_self (every indexed point a centre; "
                                "centres read in the index's cell order, no key sort)"
                                if self_q else "cm_radius_search (cell-key radix sort of the "
                                "shard's centres)"),
                       "pool": f"cm_pool_configure(keep {pool_keep >> 30} GiB, "
                               f"reserve {pool_reserve >> 30} GiB)"},
            "build_ms": {k: round(v, 3) for k, v in build_ms.items()},
            "build_detail": build_detail,
            "build_roofline": build_roof,
            "phases_ms": phase,
            "general_centres": general,
            "tile_stats": step_stats if any(step_stats.values()) else
            "tile counters are compiled into the checked library only (libcmgpu_checked.so)",
            "roofline": roofline,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if any(rsn in BAD_REASONS for rsn in clk.get("reasons", [])):
            line["clocks_warning"] = "throttle reason active during the timed region"
        emit(line)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
