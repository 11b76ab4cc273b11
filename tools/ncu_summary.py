"""Summarise ncu captures into profiles/ (run here, on the CPU box, from gpurun_out/ files)."""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__warps_active.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "smsp__inst_executed.sum", "sm__cycles_active.avg", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_bytes.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {n: (x, un) for n, un, x in zip(h, u, v)}


def stalls(rep):
    r = raw(rep)
    return {n.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(x)) for n, (x, _) in r.items()
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")
            and x not in ("", "n/a") and float(x) > 0}


def opmix(rep, nodes, nodes_per_rowstep=128):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[1], rows[2:]
    ci, si = hdr.index("Instructions Executed"), hdr.index("Source")
    import re
    ops = collections.Counter()
    for r in data:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[si].strip())
        ops[m.group(2) if m else "?"] += int(r[ci] or 0)
    steps = nodes / nodes_per_rowstep
    return {k: round(v / steps, 1) for k, v in ops.most_common(20)}


def main(rep, nodes, title, out_txt, algo_bytes):
    r = raw(rep)
    lines = ["# %s" % title, "# source: %s (ncu --set full --clock-control none)" % rep, ""]
    for k in KEYS:
        if k in r:
            lines.append("%-70s %s %s" % (k, r[k][0], r[k][1]))
    dur_ns = float(r["gpu__time_duration.sum"][0]) * (1000.0 if r["gpu__time_duration.sum"][1] == "us" else 1.0)
    rd = float(r["dram__bytes_read.sum"][0]) * (1e6 if r["dram__bytes_read.sum"][1] == "Mbyte" else 1e9 if r["dram__bytes_read.sum"][1] == "Gbyte" else 1)
    wr = float(r["dram__bytes_write.sum"][0]) * (1e6 if r["dram__bytes_write.sum"][1] == "Mbyte" else 1e9 if r["dram__bytes_write.sum"][1] == "Gbyte" else 1)
    lines += ["", "algorithmic bytes per launch (48 B x %d node-updates): %d" % (nodes, algo_bytes),
              "dram traffic per launch (read + write): %d (%.3f x algorithmic)" % (rd + wr, (rd + wr) / algo_bytes),
              "achieved under ncu (serialised, cold): %.1f GB/s algorithmic" % (algo_bytes / dur_ns),
              "", "warp stall samples: " + json.dumps(stalls(rep)),
              "", "executed warp-instructions per 128-node row step (one warp, one row): " + json.dumps(opmix(rep, nodes))]
    open(out_txt, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return rd + wr


if __name__ == "__main__":
    rep, nodes, title, out_txt = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
    traffic = main(rep, nodes, title, out_txt, 48 * nodes)
    if len(sys.argv) > 5:
        tj = sys.argv[5]
        try:
            t = json.load(open(tj))
        except Exception:
            t = {}
        key = sys.argv[6]
        t.setdefault("fast_step_kernel", {})
        t[key] = {"workload": key, "dram_bytes_per_launch": traffic, "source": rep}
        # bench.py looks up t["fast_step_kernel"] for its default workload
        if key == "cfg2_64x256x256":
            t["fast_step_kernel"] = t[key]
        json.dump(t, open(tj, "w"), indent=1)
