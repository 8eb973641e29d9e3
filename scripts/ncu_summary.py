"""Summarise ncu outputs for profiles/ (run here, on the reports gpurun brought back).
    python scripts/ncu_summary.py launches <launches.csv>
    python scripts/ncu_summary.py full <report.ncu-rep>"""
import csv, subprocess, sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            name = r[ki]
            for tag in ("TF1Op", "TF2Op", "TA1Op", "TA2Op", "A3Op", "MaskRowsOp", "ColsOp", "RowsOp", "F1Op", "F2Op", "A1Op", "A2Op"):
                if tag + "<" in name or tag + "I" in name:
                    name = f"k_pass[{tag}]"
                    break
            else:
                name = name.split("(")[0].replace("unnamed>::", "")
            d[name].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    print(f"{'kernel':45s} {'n':>5s} {'mean_us':>9s} {'total_us':>10s} {'share':>6s}")
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        print(f"{k[:45]:45s} {len(v):5d} {sum(v)/len(v)/1e3:9.1f} {sum(v)/1e3:10.1f} {sum(v)/tot*100:5.1f}%")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    print("kernel:", v[h.index("Kernel Name")][:160])
    for w in WANT:
        if w in h:
            print(f"  {w:70s} {v[h.index(w)]:>16s} {u[h.index(w)]}")
    st = [(float(v[i]), h[i]) for i in range(len(h))
          if "issue_stalled" in h[i] and "per_issue_active" in h[i] and v[i] not in ("", "n/a")]
    print("  stalls per issued instruction:",
          ", ".join("%s=%.2f" % (n.split("stalled_")[1].split("_per")[0], x) for x, n in sorted(st, reverse=True)[:8]))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
