"""The concurrency contract: a built map is immutable and may be queried by
any number of threads at once (/root/reference/proj/core/include/cheesemap/
map.hpp:50-52; include/cmgpu.h "Conventions"). Eight host threads, each on
its own CUDA stream, query ONE index at the same time — radius searches
(single-pass collect, the large-radius count + fill path, host and device
buffers), digests and kNN — and every result must equal the CPU oracle's.
ctypes releases the GIL around each C call, so the calls really overlap."""
import ctypes
import threading

import numpy as np
import pytest

from paper_2502_11602_b200 import _native
from paper_2502_11602_b200 import cheesemap as cm
from paper_2502_11602_b200 import synth
from oracle.oracle import CpuIndex

pytestmark = pytest.mark.gpu


def test_eight_threads_eight_streams_one_index():
    import torch

    cloud = synth.config_cloud(1, scale=0.02)  # 400k points, buildings included
    oracle = CpuIndex(cloud, flavor=1)
    d = torch.from_numpy(cloud).cuda()
    m = cm.Cheesemap.build(d, cm.BuildOptions(flavor=cm.Flavor.Mixed))
    rng = np.random.default_rng(7)
    jobs = []
    for t in range(8):
        q = np.ascontiguousarray(cloud[rng.choice(cloud.shape[0], 40_000 + 5000 * t, replace=False)])
        kind = ["csr", "csr_dev", "digest", "knn"][t % 4]
        r = [0.5, 1.0, 2.5, 1.0, 3.0, 1.0, 0.5, 1.5][t]
        kernel = cm.CUBE if t in (1, 4) else cm.SPHERE
        jobs.append(dict(q=q, kind=kind, r=r, kernel=kernel, k=8 + 8 * (t // 4)))
    results = [None] * len(jobs)
    errors = []
    start = threading.Barrier(len(jobs))

    def work(i):
        try:
            j = jobs[i]
            s = torch.cuda.Stream()
            start.wait()
            out = []
            for _rep in range(3):
                with torch.cuda.stream(s):
                    if j["kind"] == "csr":
                        out.append(cm.radius_search_batch(m, j["q"], j["r"], j["kernel"], stream=s))
                    elif j["kind"] == "csr_dev":
                        qd = torch.from_numpy(j["q"]).to("cuda", non_blocking=False)
                        row, cols = cm.radius_search_batch(m, qd, j["r"], j["kernel"], stream=s,
                                                           device_out=True)
                        s.synchronize()
                        out.append((row.cpu().numpy().astype(np.uint64),
                                    cols.cpu().numpy().view(np.uint32)))
                    elif j["kind"] == "digest":
                        out.append(cm.radius_digest_batch(m, j["q"], j["r"], j["kernel"], stream=s))
                    else:
                        out.append(cm.knn_batch(m, j["q"], j["k"], stream=s))
            results[i] = out
        except Exception as ex:  # noqa: BLE001
            errors.append((i, repr(ex)))

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for j, out in zip(jobs, results):
        if j["kind"] in ("csr", "csr_dev"):
            exp = oracle.radius_csr(j["q"], int(j["kernel"]), j["r"])
        elif j["kind"] == "digest":
            exp = oracle.radius(j["q"], int(j["kernel"]), j["r"])
        else:
            exp = oracle.knn(j["q"], j["k"])
        for got in out:
            assert all(np.array_equal(a, b) for a, b in zip(got, exp)), (j["kind"], j["r"])
    # per-thread timing state stays per thread: a fresh thread has none
    rc = []
    th = threading.Thread(target=lambda: rc.append(
        _native.lib().cm_get_last_query_timing(ctypes.byref(_native.QueryTimingC()))))
    th.start()
    th.join()
    assert rc == [2]  # CM_INVALID_ARGUMENT
