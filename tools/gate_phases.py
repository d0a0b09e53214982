"""Timeline of the whole-GPU fused gating path (globaltimer ns): top-k grid start /
end, routing CTA 0 start, masks staged, PDL dependency released, end.
python tools/gate_phases.py"""
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
        z = s[24]  # first top-k CTA's start
        print("B", B, "ns after the top-k grid starts: grid done", s[25] - z, "routing CTA start", s[20] - z,
              "masks staged", s[21] - z, "dependency released", s[22] - z, "end", s[23] - z, flush=True)
        st.zero_()


if __name__ == "__main__":
    main()
