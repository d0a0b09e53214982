"""Fold tools/sweep.sh output (one bench.py JSON line per config) into the committed
profiles/<round>_sweep.json table.  python tools/sweep_table.py gpurun_out/sweep.jsonl r1"""

import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    src, rnd = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "r1")
    rows = []
    for line in open(src):
        if not line.strip():
            continue
        d = json.loads(line)
        c, cpu, lam = d["config"], d["cpu_baseline"], d["lambda"]
        rows.append({
            "config": c["name"], "workload": c["workload"], "B": c["global_batch"], "G": c["ep_ranks"],
            "ratio": c["replication"], "route_us": round(d["value"], 3),
            "route_no_pdl_us": round(d["timing"]["no_pdl_us"], 3), "e2e_us": round(d["e2e"]["value"], 3),
            "cpu_port_us": round(cpu["value"], 3), "cpu_port_median_us": round((cpu.get("per_layer_us") or {}).get("median")
                                        or cpu["per_layer"]["metro_layer_us"]["median"], 3),
            "e2e_speedup_vs_cpu_port": round(cpu["value"] / d["e2e"]["value"], 3),
            "python_reference_median_us": (cpu.get("python_reference") or {}).get("median_us"),
            "lambda_metro_mean": lam["metro_mean"], "lambda_eplb_mean": lam["eplb_mean"],
            "metro_le_eplb_all": lam["metro_le_eplb_all"], "batches": lam["batches"],
            "lambda_per_physical_gpu": (lam.get("detail") or {}).get("per_physical_gpu"),
            "sm_mhz": d["clocks"]["sm_mhz"], "clock_reasons": d["clocks"]["reasons"],
            "parity_vs_gpu": cpu.get("parity_vs_gpu"),
        })
    out = {"what": ("bench.py over every BASELINE configuration (+ Zipf skew 0.5 / 2.0 of the decode batch), N=1, "
                    "one B200 (tools/sweep.sh); route = exactly-K graph-replayed us/layer over a >L2 pool (PDL), "
                    "e2e = ServedRouter host call, cpu = oracle port single thread, pinned (mean; median beside), lambda "
                    "over the bench's lambda batches (32 in round 1, 128 fresh seeds from round 2)"), "rows": rows}
    with open(os.path.join(REPO, "profiles", f"{rnd}_sweep.json"), "w") as f:
        json.dump(out, f, indent=1)
    for r in rows:
        print(f"{r['config']:18s} route {r['route_us']:6.2f}  e2e {r['e2e_us']:6.2f}  cpu {r['cpu_port_us']:6.2f}  "
              f"x{r['e2e_speedup_vs_cpu_port']:.2f}  lam {r['lambda_metro_mean']} / {r['lambda_eplb_mean']}")


if __name__ == "__main__":
    main()
