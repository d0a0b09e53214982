"""Timeline of the whole-GPU fused gating kernel's routing CTA (globaltimer ns) and
of the single-cluster variant (clock64 phases).  python tools/gate_phases.py"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import DevicePlacement, Router, _native  # noqa: E402
from paper_2512_09277_b200.placement import make_placement  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    pl = DevicePlacement(make_placement(256, 8, 1.5, 7).matrix, dev)
    L = _native.lib()
    st = torch.zeros(32, dtype=torch.int64, device=dev)
    for B in (256, 1024, 4096):
        r = Router(pl, "metro")
        sc = torch.randn((B, 256), device=dev)
        for _ in range(3):
            r.route_scores(sc, 8, whole_gpu=True)
        torch.cuda.synchronize()
        L.metro_debug_set_stamps(ctypes.c_void_p(st.data_ptr()))
        r.route_scores(sc, 8, whole_gpu=True)
        torch.cuda.synchronize()
        L.metro_debug_set_stamps(None)
        s = st.cpu().tolist()
        print("whole-GPU B", B, "topk ns", s[21] - s[20], "arrival ns", s[22] - s[21], "route+outputs ns",
              s[23] - s[22], "decide cycles", s[6] - s[3] if s[6] > s[3] else None, flush=True)


if __name__ == "__main__":
    main()
