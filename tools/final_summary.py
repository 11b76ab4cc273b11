"""Turns the files of tools/final_gpu.sh (gpurun_out/final/) into the tracked evidence under
profiles/: bench lines, range-replay summaries, per-kernel ncu summaries and traffic.json (the
DRAM bytes per node-update bench.py reports as roofline.traffic). Runs here (CPU box, needs ncu
only to read reports)."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "final")
PRO = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__cycles_active.avg", "lts__t_bytes.sum"]
NODES = 67108864


def line(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def val(x, u):
    return float(x) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3}.get(u, 1)


def range_summary(name, cid, steps, bench_json, out_name, what):
    rows = list(csv.reader(open(os.path.join(SRC, name + ".csv"))))
    d = {h: (x, u) for h, u, x in zip(rows[0], rows[1], rows[2])}
    b = line(os.path.join(SRC, bench_json))
    nu = steps * NODES
    tr = val(*d["dram__bytes_read.sum"]) + val(*d["dram__bytes_write.sum"])
    L = ["# r02 (final code): ncu RANGE replay of the whole timed region of bench.py --config %d "
         "--steps %d (NVTX range bench_timed around cb.benchmark(%d)): %s" % (cid, steps, steps, what),
         "# SC_BENCH_NVTX=1 ncu --replay-mode range --nvtx --nvtx-include bench_timed/ "
         "--clock-control none --metrics ... (tools/final_gpu.sh; source: gpurun_out/final/%s.ncu-rep)"
         % name, ""]
    for k in KEYS:
        L.append("%-70s %s %s" % (k, d[k][0], d[k][1]))
    L += ["", "node-updates in the range: %d; algorithmic bytes (48 B each): %d" % (nu, 48 * nu),
          "DRAM traffic read + write: %d = %.2f B per node-update (%.3f x algorithmic)"
          % (tr, tr / nu, tr / (48 * nu)),
          "warp-instructions per 128-node row step: %.0f"
          % (float(d["smsp__inst_executed.sum"][0]) / (nu / 128)),
          "the same command without ncu (profiles/r02_bench/%s): region %.3f ms, %.4e "
          "node-updates/s, roofline.frac %.4f" % (bench_json, b["roofline"]["region_ms"],
                                                  b["value"], b["roofline"]["frac"])]
    open(os.path.join(PRO, out_name), "w").write("\n".join(L) + "\n")
    return tr, nu


def main():
    os.makedirs(os.path.join(PRO, "r02_bench"), exist_ok=True)
    for f in os.listdir(SRC):
        if f.endswith(".json"):
            shutil.copy(os.path.join(SRC, f), os.path.join(PRO, "r02_bench", f))
    shutil.copy(os.path.join(SRC, "pytest_gpu.txt"), os.path.join(PRO, "r02_pytest_gpu.txt"))
    shutil.copy(os.path.join(SRC, "launches_cfg5_s20.csv"),
                os.path.join(PRO, "r02_launches_bench_cfg5_s20.csv"))
    shutil.copy(os.path.join(SRC, "launches_cfg5.csv"),
                os.path.join(PRO, "r02_launches_bench_cfg5.csv"))
    tj = json.load(open(os.path.join(PRO, "traffic.json")))
    for name, cid, steps, bj, out, what, key in [
        ("range_cfg5_s20", 5, 20, "cfg5_s20.json", "r02_range_bench_cfg5_s20.txt",
         "the driver's command form, 80 fast_step_kernel launches (four concurrent cloth chunks)",
         "fast_step_kernel:cfg5_4096x128x128"),
        ("range_cfg4_s20", 4, 20, "cfg4_s20.json", "r02_range_bench_cfg4_s20.txt",
         "20 whole-cloth launches of the wide-register streaming kernel",
         "fast_step_kernel:cfg4_8192x8192"),
        ("range_cfg5", 5, 300, "cfg5.json", "r02_range_bench_cfg5.txt",
         "one 12-level wavefront launch for the 2731 collider-free cloths on 100 SMs, concurrently "
         "300 plane-only streaming launches for the 1365 plane cloths on a side stream",
         "wave_kernel+fast_step_kernel:cfg5_4096x128x128")]:
        tr, nu = range_summary(name, cid, steps, bj, out, what)
        tj[key] = {"dram_bytes": tr, "node_updates": nu, "nodes": NODES, "steps": steps,
                   "source": "profiles/%s (ncu range replay of the whole timed region of "
                             "bench.py --config %d --steps %d)" % (out, cid, steps)}
    json.dump(tj, open(os.path.join(PRO, "traffic.json"), "w"), indent=1)
    # kernel summaries written on the GPU box by tools/ncu_summary.py (final_gpu.sh)
    for src, out in [("fast_cfg5_s20.txt", "r02_fast_step_chunk_cfg5_s20.txt"),
                     ("step_cfg3.txt", "r02_fast_step_cfg3.txt"),
                     ("step_cfg4.txt", "r02_fast_step_cfg4.txt"),
                     ("wave_cfg5.txt", "r02_wave_bench_cfg5.txt")]:
        shutil.copy(os.path.join(SRC, src), os.path.join(PRO, out))
    wn = 2731 * 128 * 128
    for ln in open(os.path.join(SRC, "wave_cfg5.txt")):
        if ln.startswith("dram traffic per launch"):
            tj["wave_kernel:cfg5_4096x128x128"] = {
                "dram_bytes": float(ln.split(":")[1].split("(")[0]), "nodes": wn, "steps": 300,
                "levels": 12, "node_updates": wn * 300,
                "source": "profiles/r02_wave_bench_cfg5.txt (ncu --set full of the bench's timed "
                          "wavefront launch: the 2731 collider-free cloths)"}
    json.dump(tj, open(os.path.join(PRO, "traffic.json"), "w"), indent=1)
    for f in sorted(os.listdir(os.path.join(PRO, "r02_bench"))):
        d = line(os.path.join(PRO, "r02_bench", f))
        print("%-28s steps %4s  %.4e  %8.2f us/step  frac %.4f  e2e %.3e  cpu %.3e  %s" % (
            f, d.get("steps"), d["value"], 1e3 * d.get("ms_per_step", 0),
            d.get("roofline", {}).get("frac", 0), d["e2e"]["value"],
            d.get("cpu_baseline", {}).get("value", 0), d.get("clocks", {}).get("reasons")))


if __name__ == "__main__":
    main()
