"""Per-config sweep on one GPU: device-resident queries/s for every
(config, radius, kernel) of BASELINE.json, kNN rates for config 3, and build
times, each verified against the CPU oracle on a query sample.

    python scripts/sweep.py [--configs 0,1,2,3] [--sample 2000] > sweep.json

Not the driver's bench contract (bench.py is); evidence for DESIGN.md."""
import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import CpuIndex  # noqa: E402
from paper_2502_11602_b200 import _native, synth  # noqa: E402
from paper_2502_11602_b200 import cheesemap as cm  # noqa: E402

L = _native.lib()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def timed(fn, reps=3, release=None):
    """Best of `reps` device-timed calls; `release(out)` runs after each
    call except the last, outside the timed region."""
    best = None
    for i in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
        if release is not None and i + 1 < reps:
            release(out)
    return best, out


def digest_case(m, qd, qh_sample, oracle, kernel, r, n_sample):
    """Outputs too large to materialise (TLS): per-query count + set digest."""
    nq = qd.shape[0]
    cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
    dig = torch.empty(nq, dtype=torch.int64, device="cuda")

    def run():
        cm._check(L.cm_radius_digest(m.handle, ctypes.c_void_p(qd.data_ptr()), nq, kernel, r,
                                     ctypes.c_void_p(cnt.data_ptr()),
                                     ctypes.c_void_p(dig.data_ptr()), None))

    run()
    ms, _ = timed(run, reps=2)
    c2, d2 = cm.radius_digest_batch(m, qh_sample, r, kernel)
    oc, od = oracle.radius(qh_sample, kernel, r)
    ok = bool(np.array_equal(c2, oc) and np.array_equal(d2, od))
    return dict(kernel=["sphere", "cube"][kernel], r=r, nq=nq, ms=round(ms, 3),
                qps=nq / (ms * 1e-3), nnz=int(cnt.to(torch.int64).sum().item()), mode="digest",
                verified_sample=n_sample, parity=ok)


def radius_case(m, qd, qh_sample, oracle, kernel, r, n_sample, check_all=True):
    if r >= 5.0:
        qd = qd[: qd.shape[0] // 10]  # keep the CSR (4 B x ~1000-1800 x nq) in memory
    nq = qd.shape[0]

    def run():
        csr = ctypes.c_void_p()
        cm._check(L.cm_radius_search(m.handle, ctypes.c_void_p(qd.data_ptr()), nq, kernel, r,
                                     None, ctypes.byref(csr)))
        return csr

    run_ms = None
    for _ in range(2):  # warm
        L.cm_csr_free(run())
    ms, csr = timed(run, release=L.cm_csr_free)
    t = _native.last_query_timing()
    # the timed CSR itself, every row: sorted, and (count, digest) equal to
    # the digest pass's (which the oracle checks on the sample below)
    full_ok = None
    if check_all:
        rp, cp = ctypes.c_void_p(), ctypes.c_void_p()
        cm._check(L.cm_csr_info(csr, None, None, ctypes.byref(rp), ctypes.byref(cp)))
        c1 = torch.empty(nq, dtype=torch.int32, device="cuda")
        d1 = torch.empty(nq, dtype=torch.int64, device="cuda")
        bad = ctypes.c_uint64()
        cm._check(L.cm_csr_digest(rp, cp, nq, ctypes.c_void_p(c1.data_ptr()),
                                  ctypes.c_void_p(d1.data_ptr()), ctypes.byref(bad), None))
        L.cm_csr_free(csr)
        c2 = torch.empty_like(c1)
        d2 = torch.empty_like(d1)
        cm._check(L.cm_radius_digest(m.handle, ctypes.c_void_p(qd.data_ptr()), nq, kernel, r,
                                     ctypes.c_void_p(c2.data_ptr()),
                                     ctypes.c_void_p(d2.data_ptr()), None))
        full_ok = bool(bad.value == 0 and torch.equal(c1, c2) and torch.equal(d1, d2))
        del c1, d1, c2, d2
    else:
        L.cm_csr_free(csr)
    # verification on a sample: counts + digests vs the oracle
    cnt, dig = cm.radius_digest_batch(m, qh_sample, r, kernel)
    ocnt, odig = oracle.radius(qh_sample, kernel, r)
    ok = bool(np.array_equal(cnt, ocnt) and np.array_equal(dig, odig))
    tested = torch.zeros(nq, dtype=torch.int64, device="cuda")
    cm._check(L.cm_radius_count(m.handle, ctypes.c_void_p(qd.data_ptr()), nq, kernel, r, None,
                                ctypes.c_void_p(tested.data_ptr()), None))
    alg = 24 * int(tested.sum().item())
    free_b, total_b = torch.cuda.mem_get_info()
    log(f"    two_pass={t['two_pass']} nnz={t['nnz']} free={free_b / 1e9:.1f} GB")
    return dict(kernel=["sphere", "cube"][kernel], r=r, nq=nq, ms=round(ms, 3),
                qps=nq / (ms * 1e-3), nnz=int(t["nnz"]), two_pass=int(t["two_pass"]),
                phases={k: round(t[k], 3) for k in ("order_ms", "pass1_ms", "scan_ms", "pass2_ms")},
                alg_gb=round(alg / 1e9, 2), frac_pass1=round(alg / (t["pass1_ms"] * 1e-3) / 6542.1e9, 3),
                verified_sample=n_sample, parity=ok, csr_all_rows_ok=full_ok)


def knn_case(m, qd, qh_sample, oracle, k):
    nq = qd.shape[0]
    idx = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    d2 = torch.empty((nq, k), dtype=torch.float64, device="cuda")

    def run():
        cm._check(L.cm_knn(m.handle, ctypes.c_void_p(qd.data_ptr()), nq, k,
                           ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(d2.data_ptr()), None))

    run()
    ms, _ = timed(run)
    gi, gd = cm.knn_batch(m, qh_sample, k)
    oi, od, prk, pa2 = oracle.knn(qh_sample, k, stats=True)
    ok = bool(np.array_equal(gi, oi) and np.array_equal(gd, od))
    # SURVEY 8d kNN bytes: 24 B x points_tested(kernel_search(c, r_k)), r_k
    # the exact k-th distance — estimated from the oracle on the sample
    alg = 24.0 * float(prk.mean()) * nq
    return dict(k=k, nq=nq, ms=round(ms, 3), qps=nq / (ms * 1e-3), parity=ok,
                alg_gb_est=round(alg / 1e9, 2), frac_est=round(alg / (ms * 1e-3) / 6542.1e9, 3),
                ref_alg2_tested_mean=round(float(pa2.mean()), 1),
                rk_tested_mean=round(float(prk.mean()), 1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,1,2,3")
    ap.add_argument("--sample", type=int, default=1000)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--flavors", default=None, help="subset, e.g. mixed")
    ap.add_argument("--radii", default=None, help="subset, e.g. 2.5,5")
    ap.add_argument("--kernels", default=None, help="subset, e.g. 0")
    a = ap.parse_args()
    # this process owns the GPU (as the bench does): keep 3/4 of HBM cached in
    # the library's pool and reserve 32 GiB, so the large CSRs' allocations do
    # not map fresh memory inside the timed calls
    total_mem = torch.cuda.get_device_properties(0).total_memory
    if hasattr(L, "cm_pool_configure"):
        cm.pool_configure(0, int(total_mem * 0.75), min(32 << 30, int(total_mem * 0.2)))
    out = {"gpu": torch.cuda.get_device_name(0), "results": []}
    cfgs = [int(c) for c in a.configs.split(",")]
    plan = {
        0: dict(flavors=["dense"], cell=1.0, radii=[1.0], kernels=[0, 1], ks=[]),
        1: dict(flavors=["mixed", "sparse"], cell=1.0, radii=[0.5, 1.0, 2.5, 5.0], kernels=[0, 1],
                ks=[]),
        2: dict(flavors=["mixed"], cell=0.25, radii=[0.05, 0.1, 0.25], kernels=[0], ks=[],
                digest=True),
        3: dict(flavors=["mixed"], cell=1.0, radii=[], kernels=[], ks=[8, 16, 32, 64]),
        # 200M points on one GPU; r = 2.5 as digests (its CSR would be ~170 GB)
        4: dict(flavors=["mixed"], cell=1.0, radii=[1.0, 2.5], kernels=[0], ks=[],
                digest_radii=[2.5]),
    }
    fl = {"dense": 0, "sparse": 1, "mixed": 2}
    for c in cfgs:
        t0 = time.perf_counter()
        cloud = synth.config_cloud(c, a.scale)
        q = synth.config_queries(c, cloud)
        log(f"config {c}: {cloud.shape[0]} points, {q.shape[0]} queries "
            f"({time.perf_counter() - t0:.1f}s)")
        p = dict(plan[c])
        if a.flavors:
            p["flavors"] = [f for f in p["flavors"] if f in a.flavors.split(",")]
        if a.radii:
            p["radii"] = [r for r in p["radii"] if r in [float(x) for x in a.radii.split(",")]]
        if a.kernels:
            p["kernels"] = [k for k in p["kernels"] if k in [int(x) for x in a.kernels.split(",")]]
        dc = torch.from_numpy(cloud).cuda()
        qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
        rng = np.random.default_rng(c)
        samp = np.ascontiguousarray(q[rng.choice(q.shape[0], min(a.sample, q.shape[0]),
                                                 replace=False)])
        oracle = CpuIndex(cloud, flavor=1, cell=(p["cell"],) * 3)
        for f in p["flavors"]:
            opts = cm.BuildOptions(flavor=cm.Flavor(fl[f]), cell=cm.CellSize.uniform(p["cell"]))
            builds = []
            for _ in range(3):
                m = cm.Cheesemap.build(dc, opts)
                builds.append(m.build_timing()["total_ms"])
            entry = {"config": c, "flavor": f, "n_points": int(cloud.shape[0]),
                     "build_ms": round(min(builds), 3), "radius": [], "knn": []}
            for r in p["radii"]:
                for kern in p["kernels"]:
                    fn = (digest_case if p.get("digest") or r in p.get("digest_radii", ())
                          else radius_case)
                    res = fn(m, qd, samp, oracle, kern, r, samp.shape[0])
                    log(f"  cfg{c} {f} {res['kernel']} r={r}: {res['qps'] / 1e6:.1f} M q/s "
                        f"parity={res['parity']} all_rows={res.get('csr_all_rows_ok')} phases={res.get('phases', res.get('mode'))}")
                    entry["radius"].append(res)
            for k in p["ks"]:
                res = knn_case(m, qd, samp, oracle, k)
                log(f"  cfg{c} {f} knn k={k}: {res['qps'] / 1e6:.2f} M q/s parity={res['parity']} "
                    f"frac_est={res['frac_est']} tested(r_k)={res['rk_tested_mean']}")
                entry["knn"].append(res)
            out["results"].append(entry)
            del m
        del oracle, dc, qd
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
