"""clock64 phase stamps (CTA 0) of the fused route + layout kernel vs routing
alone: where the layout's extra time goes.  python tools/fused_phase.py"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, DispatchLayout, Router, _native  # noqa: E402
from paper_2512_09277_b200.placement import gen_zipf_topk, make_placement  # noqa: E402

COLD = os.environ.get("COLD", "1") == "1"  # 0: no L2 flush before the stamped launch (code L2-warm)
SHAPES = {"q30": (128, 8, 1.5, 256), "ds_b64": (256, 8, 1.5, 64), "ds": (256, 8, 1.5, 1024),
          "ds_b8192": (256, 8, 1.5, 8192)}


def main():
    dev = torch.device("cuda", 0)
    L = _native.lib()
    st = torch.zeros(32, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    res = {}
    for name, (n, g, ratio, B) in SHAPES.items():
        pl = DevicePlacement(make_placement(n, g, ratio, 7).matrix, dev)
        ids = torch.from_numpy(gen_zipf_topk(n, 8, B, 1.2, 1000, popularity_seed=7)).to(dev)
        r, dl = Router(pl, "metro"), DispatchLayout(pl)
        out, lo = r.alloc(B * 8, top_k=8), dl.alloc(B * 8, 8)
        for variant, fn in (("route", lambda: r.route(ids, out=out)),
                            ("fused", lambda: dl.route_metro(ids, out=out, layout_out=lo))):
            for _ in range(5):
                fn()
            rows = []
            for _ in range(5):
                st.zero_()
                L.metro_debug_set_stamps(ctypes.c_void_p(st.data_ptr()))
                if COLD:
                    flush.zero_()
                fn()
                torch.cuda.synchronize()
                L.metro_debug_set_stamps(None)
                rows.append(st.cpu().tolist())
            s = sorted(rows, key=lambda x: x[7] - x[0])[2]  # the median launch
            d = {"stage": s[1] - s[0], "hist": s[2] - s[1], "rowsum": s[3] - s[2], "to_greedy": s[5] - s[3],
                 "greedy": s[6] - s[5], "after_greedy": s[7] - s[6], "total": s[7] - s[0]}
            if variant == "fused":
                d.update({"walk_start_after_greedy_start": s[30] - s[5], "walk_end_after_greedy_start": s[26] - s[5], "walk_prefix_end": s[29] - s[5],
                          "tail_barrier": s[28] - s[6], "outputs": s[7] - s[28]})
            res[f"{name}/{variant}"] = d
            print(name, variant, d, flush=True)
    with open(f"gpurun_out/fused_phase_{'cold' if COLD else 'warm'}.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
