"""Turn the ncu artefacts of scripts/gpu_profiles.sh (gpurun_out/) into the
committed summaries: profiles/<tag>_launches.csv, <tag>_ncu_metrics.json,
ncu_traffic.json (read by bench.py for roofline.traffic)."""
import collections
import csv
import json
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
launches = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/launches_all.csv"
suffix = sys.argv[3] if len(sys.argv) > 3 else ""  # full_<kernel><suffix>.ncu-rep
rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
hdr = rows[0]
ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
out = [["launch_id", "kernel", "gpu__time_duration_ns"]]
agg = collections.defaultdict(list)
for r in rows[1:]:
    name = r[ki].split("(")[0]
    out.append([r[ii], name, r[vi].replace(",", "")])
    agg[name].append(float(r[vi].replace(",", "")))
with open(f"profiles/{tag}_launches.csv", "w", newline="") as f:
    csv.writer(f).writerows(out)
print("launch list (mean us):")
for k, v in agg.items():
    print(f"  {k[:60]:60s} n={len(v):3d} {sum(v) / len(v) / 1e3:8.2f}")


def raw(k):
    txt = subprocess.run(["ncu", "-i", f"gpurun_out/full_{k}{suffix}.ncu-rep", "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(txt.splitlines()))
    return {h: (v, u) for h, v, u in zip(rr[0], rr[2], rr[1])}


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
summ, traffic = {}, {}
for k in ["hstu_fwd", "hstu_bwd_dkv", "hstu_bwd_dq"]:
    m = raw(k)
    val = lambda n: float(m[n][0].replace(",", "")) * SCALE.get(m[n][1], 1)  # noqa: E731
    rd, wr, dur = val("dram__bytes_read.sum"), val("dram__bytes_write.sum"), val("gpu__time_duration.sum")
    stalls = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                      float(v[0])) for h, v in m.items() if h.startswith("smsp__average_warps_issue_stalled_")),
                    key=lambda x: -x[1])[:4]
    summ[k] = {"duration_us": dur * 1e6, "dram_read_MB": rd / 1e6, "dram_write_MB": wr / 1e6,
               "tensor_pipe_active_pct": float(m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"][0]),
               "xu_pipe_pct": float(m["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"][0]),
               "issue_active_pct": float(m["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
               "sm_clock_ghz": float(m["sm__cycles_elapsed.avg.per_second"][0]),
               "top_stalls": stalls}
    traffic[k] = rd + wr
json.dump(summ, open(f"profiles/{tag}_ncu_metrics.json", "w"), indent=1)
json.dump({"fwd": traffic["hstu_fwd"], "bwd": traffic["hstu_bwd_dkv"] + traffic["hstu_bwd_dq"],
           "per_kernel_bytes": traffic,
           "source": f"ncu --set full --clock-control none, one launch each (profiles/{tag}_ncu_summary.md)"},
          open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(summ, indent=1))
