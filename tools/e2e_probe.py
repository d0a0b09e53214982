"""Where the end-to-end (host buffers) routing time goes: Python/ctypes call,
kernel device time in zero-copy vs copy mode, synchronisation."""

import ctypes
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, HostRouter, Router, ServedRouter, _native  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402


def tmed(fn, n=2000):
    for _ in range(50):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6, statistics.mean(ts) * 1e6


def main():
    dev = torch.device("cuda", 0)
    L = _native.lib()
    A = make_placement(256, 8, 1.5, 7).matrix
    pl = DevicePlacement(A, dev)
    ids = torch.from_numpy(gen_zipf_topk(256, 8, 1024, 1.2, 1000, popularity_seed=7).reshape(-1).copy()).pin_memory()
    pr = torch.empty(8192, dtype=torch.int32).pin_memory()
    res = {}
    res["ctypes_noop_us"] = tmed(lambda: L.metro_abi_version())
    for zc in (True, False):
        hr = HostRouter(pl, 8192, zero_copy=zc)
        res[f"host_call_{'zc' if zc else 'copy'}_us"] = tmed(lambda: hr(ids, pr))
        # device time of the same sequence (events on the router's stream)
        s = hr.stream
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        dts = []
        for _ in range(200):
            e0.record(s)
            hr(ids, pr)
            e1.record(s)
            torch.cuda.synchronize()
            dts.append(e0.elapsed_time(e1) * 1e3)
        res[f"device_{'zc' if zc else 'copy'}_us"] = statistics.median(dts)
    with ServedRouter(pl, 8192) as sr:
        sr.ids.numpy()[:] = ids.numpy()
        res["served_us"] = tmed(lambda: sr.run(8192), n=20000)
        res["served_launches"] = sr.launches
        # the caller rewrites its batch before every call (dirty lines in the CPU
        # caches when the GPU reads them)
        import numpy as np
        src = [np.roll(ids.numpy(), j) for j in range(8)]
        dst = sr.ids.numpy()
        per = []
        for j in range(5000):
            dst[:] = src[j % 8]
            t0 = time.perf_counter()
            sr.run(8192)
            per.append(time.perf_counter() - t0)
        res["served_rewritten_us"] = (statistics.median(per) * 1e6, statistics.mean(per) * 1e6)
    r = Router(pl, "metro")
    d_ids = ids.to(dev)
    out = r.alloc(8192, top_k=8)
    res["device_launch_sync_us"] = tmed(lambda: (r.route(d_ids, out=out), torch.cuda.current_stream().synchronize()))
    st = torch.cuda.Stream()
    res["empty_sync_us"] = tmed(lambda: st.synchronize())
    for k, v in res.items():
        print(k, v)


if __name__ == "__main__":
    main()
