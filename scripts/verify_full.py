"""Full-population parity at BASELINE sizes: for EVERY query of a config,
the GPU's per-query (count, digest) against the multithreaded CPU oracle.

    python scripts/verify_full.py [--configs 1,2,3,4] [--out profiles/r02/verify_full.json]

The reference's acceptance test compares every case, not a sample
(/root/reference/proj/tests/acceptance.cpp:79-137); this does the same for
kernel_search (search.hpp:102-127) at the configs' full sizes:

  * the oracle (oracle/cheesemap_oracle.cpp, test infrastructure) answers
    every query on all host threads: neighbour count and the set digest
    sum(splitmix64(handle)) mod 2^64 — order-free, so no sort on the CPU;
  * the GPU answers the same queries twice, through independent paths:
      - the DIGEST pass (cm_radius_digest), and
      - the product CSR (cm_radius_search / cm_radius_search_self, in
        query chunks when the CSR would not fit), reduced by cm_csr_digest to
        (count, digest, rows not strictly ascending);
    both are compared with the oracle for every query. A digest collision
    would need two different handle sets with equal 64-bit mixed sums.
  * kNN (config 3): cm_knn for all centres of the stream; the oracle's
    (handle, d^2) rows for the first --knn-sample centres, compared exactly.

Every case records the number of queries checked, the mismatches (0 is the
bar), the oracle's thread count and both sides' times. The chunked CSR
calls are timed too (device events), so the large-radius cases report the
rate over the whole query population.
"""
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

FL = {"dense": 0, "sparse": 1, "mixed": 2}
KN = {0: "sphere", 1: "cube"}

# config -> flavours, cell, radii, kernels, self (every point a query)
PLAN = {
    0: dict(flavors=["dense", "sparse", "mixed"], cell=1.0, radii=[1.0], kernels=[0, 1], self=False),
    1: dict(flavors=["sparse", "mixed"], cell=1.0, radii=[0.5, 1.0, 2.5, 5.0], kernels=[0, 1],
            self=True),
    2: dict(flavors=["mixed"], cell=0.25, radii=[0.05, 0.1, 0.25], kernels=[0], self=False),
    3: dict(flavors=["mixed"], cell=1.0, ks=[8, 16, 32, 64]),
    4: dict(flavors=["sparse"], cell=1.0, radii=[1.0, 2.5], kernels=[0], self=True),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def L():
    return _native.lib()


def _vp(t):
    return ctypes.c_void_p(t.data_ptr())


class Oracle:
    """The CPU restatement over the whole cloud, all host threads."""

    def __init__(self, cloud, cell, threads):
        t0 = time.perf_counter()
        self.idx = CpuIndex(cloud, flavor=1, cell=(cell,) * 3)
        self.build_s = time.perf_counter() - t0
        self.threads = threads or os.cpu_count() or 1

    def radius(self, q, kernel, r):
        t0 = time.perf_counter()
        c, d = self.idx.radius(q, kernel, r, threads=self.threads)
        return c, d, time.perf_counter() - t0


def device_events():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def compare(name, gc, gd, oc, od, extra_bad=0):
    """gc/gd: device tensors (int32 / int64); oc/od: host oracle arrays."""
    tc = torch.from_numpy(oc.view(np.int32)).to(gc.device)
    td = torch.from_numpy(od.view(np.int64)).to(gd.device)
    bad = (gc != tc) | (gd != td)
    nbad = int(bad.sum().item())
    first = []
    if nbad:
        idx = torch.nonzero(bad).flatten()[:5].cpu().tolist()
        first = [dict(q=i, gpu=(int(gc[i]), int(gd[i])), oracle=(int(oc[i]), int(od[i])))
                 for i in idx]
        log(f"    MISMATCH {name}: {nbad} queries, first {first}")
    return dict(mismatches=nbad + int(extra_bad), first=first)


def gpu_digest(m, qd, nq, kernel, r):
    cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
    dig = torch.empty(nq, dtype=torch.int64, device="cuda")
    e0, e1 = device_events()
    e0.record()
    qp = _vp(qd) if qd is not None else None
    cm._check(L().cm_radius_digest(m.handle, qp, nq, kernel, r, _vp(cnt), _vp(dig), None))
    e1.record()
    e1.synchronize()
    return cnt, dig, e0.elapsed_time(e1)


def csr_digest(csr, nq, cnt_out, dig_out, off):
    rp, cp = ctypes.c_void_p(), ctypes.c_void_p()
    cm._check(L().cm_csr_info(csr, None, None, ctypes.byref(rp), ctypes.byref(cp)))
    bad = ctypes.c_uint64()
    cm._check(L().cm_csr_digest(rp, cp, nq, ctypes.c_void_p(cnt_out.data_ptr() + 4 * off),
                                ctypes.c_void_p(dig_out.data_ptr() + 8 * off), ctypes.byref(bad),
                                None))
    return int(bad.value)


def gpu_csr(m, qd, nq, kernel, r, counts_hint, budget, self_q):
    """The product CSR for every query, in chunks of <= `budget` neighbours
    (one call when it fits). Returns per-query (count, digest) of the CSR as
    device tensors, unsorted-row total, device ms summed over the calls, and
    the chunk count."""
    cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
    dig = torch.empty(nq, dtype=torch.int64, device="cuda")
    cum = torch.cumsum(counts_hint.to(torch.int64), 0)
    total = int(cum[-1].item()) if nq else 0
    bounds = [0]
    if total > budget:
        # chunk ends where the running neighbour count crosses k * budget
        marks = torch.arange(budget, total, budget, device="cuda", dtype=torch.int64)
        ends = torch.searchsorted(cum, marks).cpu().tolist()
        for e in ends:
            e = max(e, bounds[-1] + 1)
            if e < nq:
                bounds.append(e)
    bounds.append(nq)
    ms, unsorted = 0.0, 0
    for a, b in zip(bounds[:-1], bounds[1:]):
        csr = ctypes.c_void_p()
        e0, e1 = device_events()
        e0.record()
        if self_q and a == 0 and b == nq:
            cm._check(L().cm_radius_search_self(m.handle, kernel, r, None, ctypes.byref(csr)))
        else:
            qp = ctypes.c_void_p(qd.data_ptr() + 24 * a)
            cm._check(L().cm_radius_search(m.handle, qp, b - a, kernel, r, None,
                                           ctypes.byref(csr)))
        e1.record()
        e1.synchronize()
        ms += e0.elapsed_time(e1)
        unsorted += csr_digest(csr, b - a, cnt, dig, a)
        L().cm_csr_free(csr)
    return cnt, dig, unsorted, ms, len(bounds) - 1


def radius_cases(cfg, cloud, q, qd, oracle, plan, budget, only_r=None, only_k=None,
                 only_f=None):
    out = []
    nq = q.shape[0]
    dc = torch.from_numpy(cloud).cuda()
    for f in plan["flavors"]:
        if only_f and f not in only_f:
            continue
        opts = cm.BuildOptions(flavor=cm.Flavor(FL[f]), cell=cm.CellSize.uniform(plan["cell"]))
        m = cm.Cheesemap.build(dc, opts)
        for r in plan["radii"]:
            if only_r and r not in only_r:
                continue
            for k in plan["kernels"]:
                if only_k is not None and k not in only_k:
                    continue
                oc, od, ot = oracle.radius(q, k, r)
                gc, gd, dms = gpu_digest(m, qd, nq, k, r)
                res_d = compare(f"cfg{cfg} {f} {KN[k]} r={r} digest", gc, gd, oc, od)
                cc, cd, uns, cms, chunks = gpu_csr(m, qd, nq, k, r, gc, budget, plan["self"])
                res_c = compare(f"cfg{cfg} {f} {KN[k]} r={r} csr", cc, cd, oc, od, uns)
                entry = dict(config=cfg, flavor=f, kernel=KN[k], r=r, queries=nq,
                             neighbours=int(oc.astype(np.int64).sum()),
                             oracle_threads=oracle.threads, oracle_s=round(ot, 2),
                             digest_pass=dict(res_d, ms=round(dms, 3)),
                             csr=dict(res_c, unsorted_rows=uns, ms=round(cms, 3), chunks=chunks,
                                      qps=round(nq / (cms * 1e-3), 1),
                                      call=("cm_radius_search_self" if plan["self"] and chunks == 1
                                            else "cm_radius_search")))
                entry["ok"] = res_d["mismatches"] == 0 and res_c["mismatches"] == 0
                log(f"  cfg{cfg} {f} {KN[k]} r={r}: {nq} queries, digest mism "
                    f"{res_d['mismatches']}, csr mism {res_c['mismatches']} (unsorted {uns}, "
                    f"{chunks} chunks, {nq / (cms * 1e-3) / 1e6:.1f} M q/s), oracle {ot:.1f}s")
                out.append(entry)
                del gc, gd, cc, cd
        del m
        torch.cuda.empty_cache()
    del dc
    return out


def knn_cases(cloud, q, oracle, ks, sample):
    out = []
    dc = torch.from_numpy(cloud).cuda()
    qd = torch.from_numpy(q).cuda()
    nq = q.shape[0]
    m = cm.Cheesemap.build(dc, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    qs = np.ascontiguousarray(q[:sample])
    for k in ks:
        idx = torch.empty((nq, k), dtype=torch.int32, device="cuda")
        d2 = torch.empty((nq, k), dtype=torch.float64, device="cuda")
        e0, e1 = device_events()
        e0.record()
        cm._check(L().cm_knn(m.handle, _vp(qd), nq, k, _vp(idx), _vp(d2), None))
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        t0 = time.perf_counter()
        oi, od = oracle.idx.knn(qs, k, threads=oracle.threads)
        ot = time.perf_counter() - t0
        gi = idx[:sample].cpu().numpy().view(np.uint32)
        gdd = d2[:sample].cpu().numpy()
        bad_rows = int(np.count_nonzero(np.any((gi != oi) | (gdd.view(np.int64) != od.view(np.int64)),
                                               axis=1)))
        out.append(dict(config=3, k=k, queries=nq, checked=int(qs.shape[0]), mismatches=bad_rows,
                        oracle_threads=oracle.threads, oracle_s=round(ot, 2), ms=round(ms, 3),
                        qps=round(nq / (ms * 1e-3), 1), ok=bad_rows == 0,
                        compare="handles and fp64 d^2 bit-exact, order (d^2, handle)"))
        log(f"  cfg3 knn k={k}: {qs.shape[0]} of {nq} centres checked, {bad_rows} mismatching "
            f"rows; GPU {nq / (ms * 1e-3) / 1e6:.1f} M q/s; oracle {ot:.1f}s")
        del idx, d2
    del m, dc, qd
    torch.cuda.empty_cache()
    return out


def run(configs, threads=0, budget=6_000_000_000, knn_sample=500_000, only_r=None, only_k=None,
        only_f=None, scale=1.0):
    res = {"gpu": torch.cuda.get_device_name(0), "host_threads": os.cpu_count(), "cases": []}
    for c in configs:
        t0 = time.perf_counter()
        cloud = synth.config_cloud(c, scale)
        plan = PLAN[c]
        log(f"config {c}: {cloud.shape[0]} points ({time.perf_counter() - t0:.1f}s)")
        oracle = Oracle(cloud, plan["cell"], threads)
        log(f"  oracle built in {oracle.build_s:.1f}s ({oracle.threads} query threads)")
        if c == 3:
            q = synth.config_queries(3, cloud)
            res["cases"] += knn_cases(cloud, q, oracle, plan["ks"], knn_sample)
        else:
            q = synth.config_queries(c, cloud)
            qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
            res["cases"] += radius_cases(c, cloud, q, qd, oracle, plan, budget, only_r, only_k,
                                         only_f)
            del qd
        del oracle
        torch.cuda.empty_cache()
    res["all_ok"] = all(e["ok"] for e in res["cases"])
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--budget", type=float, default=6e9, help="neighbours per CSR call")
    ap.add_argument("--knn-sample", type=int, default=5_000_000)
    ap.add_argument("--radii", default=None)
    ap.add_argument("--kernels", default=None)
    ap.add_argument("--flavors", default=None)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    total = torch.cuda.get_device_properties(0).total_memory
    cm.pool_configure(0, int(total * 0.75), 0)
    res = run([int(x) for x in a.configs.split(",")], a.threads, int(a.budget), a.knn_sample,
              [float(x) for x in a.radii.split(",")] if a.radii else None,
              [int(x) for x in a.kernels.split(",")] if a.kernels else None,
              a.flavors.split(",") if a.flavors else None, a.scale)
    txt = json.dumps(res, indent=1)
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        with open(a.out, "w") as f:
            f.write(txt)
    print(json.dumps({"all_ok": res["all_ok"], "cases": len(res["cases"])}))


if __name__ == "__main__":
    main()
