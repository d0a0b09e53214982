"""Per-CTA timeline of one K3 grouped-GEMM launch (globaltimer stamps at start /
end of every persistent CTA): how much of the launch is the tail of the last
CTAs.  python tools/k3_tail_probe.py [bf16|fp8] [gate_up|down]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_09277_b200 import _native  # noqa: E402
import k3_profile_target  # noqa: E402


def main():
    L = _native.lib()
    st = torch.zeros(2 * 148, dtype=torch.int64, device="cuda")
    for rep in range(3):
        L.moe_debug_set_stamps(ctypes.c_void_p(st.data_ptr()) if rep == 2 else None)
        k3_profile_target.main()
    L.moe_debug_set_stamps(None)
    s = st.cpu().numpy().reshape(-1, 2)
    s = s[s[:, 0] > 0]  # CTAs of the launch (the balanced grid may use fewer than 148)
    print("CTAs:", len(s))
    t0 = s[:, 0].min()
    start, end = (s[:, 0] - t0) / 1e3, (s[:, 1] - t0) / 1e3
    q = np.percentile(end, [0, 10, 50, 90, 100])
    print("start us: max %.2f" % start.max())
    print("end us: min %.2f p10 %.2f p50 %.2f p90 %.2f max %.2f" % tuple(q))
    print("tail (max - p50) / max = %.3f; mean CTA busy / max = %.3f" % ((q[4] - q[2]) / q[4], np.mean(end - start) / q[4]))


if __name__ == "__main__":
    main()
