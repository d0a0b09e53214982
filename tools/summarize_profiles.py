"""Turn the ncu captures in gpurun_out/ (tools/make_profiles.sh) into committed
summaries under profiles/ (run in the build container, where ncu can import).

    python tools/summarize_profiles.py r1
"""

import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.environ.get("PROFILE_SRC") or os.path.join(REPO, "gpurun_out")
DST = os.environ.get("PROFILE_DST") or os.path.join(REPO, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__cluster_dim_x", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "lts__t_bytes.sum",
    # where the DRAM reads come from: the SM's data path (ids, masks) vs the rest (instruction /
    # constant fetch on a flushed cache)
    "dram__sectors_read.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS or h.startswith("launch__") and h in KEYS:
            res[h] = (v, u)
    res["kernel"] = (vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?", "")
    return res


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return f * scale


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r1"
    os.makedirs(DST, exist_ok=True)
    traffic = {}
    for name, rep in (("metro", "metro_full.ncu-rep"), ("moe_gemm", "moe_full.ncu-rep"),
                      ("moe_gemm_fp8", "moe_fp8_full.ncu-rep"), ("moe_gemm_down", "moe_down_full.ncu-rep"),
                      ("moe_gemm_fp8_down", "moe_fp8_down_full.ncu-rep"),
                      ("gate", "gate_full.ncu-rep"), ("gate_route", "gate_route_full.ncu-rep"),
                      ("dispatch", "dispatch_full.ncu-rep"),
                      ("exchange", "exchange_full.ncu-rep"), ("fused_route_layout", "fused_full.ncu-rep"),
                      ("metro_cache_control_none", "metro_cc_none_full.ncu-rep")):
        path = os.path.join(SRC, rep)
        if not os.path.exists(path):
            continue
        r = raw(path)
        with open(os.path.join(DST, f"{rnd}_{name}_ncu_full.txt"), "w") as f:
            f.write(f"# ncu --set full summary ({rep}); kernel {r.get('kernel', ('?',))[0]}\n")
            for k in KEYS:
                if k in r:
                    f.write(f"{k:70s} {r[k][0]:>16s} {r[k][1]}\n")
        if "dram__bytes_read.sum" in r:
            t = to_bytes(*r["dram__bytes_read.sum"]) + to_bytes(*r.get("dram__bytes_write.sum", ("0", "byte")))
            traffic[name] = t
    if "metro" in traffic:
        with open(os.path.join(DST, "ncu_traffic.json"), "w") as f:
            json.dump({"ds": traffic["metro"], "source": f"{rnd}_metro_ncu_full.txt (dram read+write bytes, "
                       "one launch, DeepSeek-V3 shape B=1024)", "moe_gemm": traffic.get("moe_gemm")}, f, indent=1)
    def launch_table(path, title):
        rows = [r for r in csv.reader(open(path)) if len(r) > 5]
        hdr = rows[0]
        kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
        tot = {}
        for r in rows[1:]:
            if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
                continue
            k = r[kn].split("(")[0][:60]
            v = float(r[mv].replace(",", ""))
            n, t = tot.get(k, (0, 0.0))
            tot[k] = (n + 1, t + v)
        lines = [title, "# cold-cache, serialised launches: compare SHARES, not absolute times (ns)"]
        allt = sum(t for _, t in tot.values()) or 1.0
        for k, (n, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
            lines.append(f"{k:62s} launches {n:5d}  mean {t / n:10.2f}  share {100 * t / allt:5.1f}%")
        return lines

    out = []
    lp = os.path.join(SRC, "launches.csv")
    if os.path.exists(lp):
        out += launch_table(lp, "# ncu --metrics gpu__time_duration.sum --clock-control none -k regex:metro_ids_kernel "
                                "(bench.py --steps 256: the timed region launches only this kernel)")
    la = os.path.join(SRC, "launches_all.csv")
    if os.path.exists(la):
        out += [""] + launch_table(la, "# same command, first 400 launches of any kernel (incl. the bench's "
                                       "one-time pool construction before the timed region)")
    if out:
        with open(os.path.join(DST, f"{rnd}_launches_summary.txt"), "w") as f:
            f.write("\n".join(out) + "\n")
    print("wrote", sorted(os.listdir(DST)))


if __name__ == "__main__":
    main()
