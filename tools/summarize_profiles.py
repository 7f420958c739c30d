#!/usr/bin/env python
"""Write the round's profile summaries under profiles/ from gpurun_out/ captures.
usage: python tools/summarize_profiles.py ROUND CFG   (e.g. r01 S7)"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def ncu_csv(args):
    out = subprocess.run(["ncu", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rnd, cfg):
    g = os.path.join(ROOT, "gpurun_out")
    pdir = os.path.join(ROOT, "profiles")
    os.makedirs(pdir, exist_ok=True)
    # 1. launch list of the bench command (cold-cache, serialised: compare shares)
    lpath = os.path.join(g, f"launches_{cfg}.csv")
    if os.path.exists(lpath):
        import launch_summary
        buf = io.StringIO()
        sys.stdout, old = buf, sys.stdout
        try:
            launch_summary.main(lpath)
        finally:
            sys.stdout = old
        with open(os.path.join(pdir, f"{rnd}_launches_{cfg}.txt"), "w") as f:
            f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, bench.py --config {cfg} "
                    "--steps 4 --warmup 3, launches inside the timed NVTX range\n")
            f.write(buf.getvalue())
    # 2. full capture of k_decode: key metrics + warp stalls + per-phase source summary
    rep = os.path.join(g, f"prof_dec_{cfg}.ncu-rep")
    if os.path.exists(rep):
        rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
        hdr, val = rows[0], rows[2] if len(rows) > 2 else rows[1]
        m = dict(zip(hdr, val))
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
                "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
                "launch__registers_per_thread", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"]
        lines = [f"# ncu --set full --import-source on --clock-control none, one k_decode launch "
                 f"({cfg}, all layers of one token; caches flushed by ncu before the launch)"]
        for k in keys:
            if k in m:
                lines.append(f"{k:80s} {m[k]}")
        rd = float(m.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
        wr = float(m.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
        unit_r = [h for h in hdr if h == "dram__bytes_read.sum"]
        src = subprocess.run(["bash", "-c", f"ncu -i {rep} --page source --csv --kernel-name regex:k_decode "
                              f"--print-source cuda,sass 2>/dev/null | python {ROOT}/tools/src_hot.py 25 stall"],
                             capture_output=True, text=True).stdout
        lines.append("\n# source lines by warp-stall samples (%s) and executed instructions (%i)")
        lines.append(src)
        with open(os.path.join(pdir, f"{rnd}_ncu_k_decode_{cfg}.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")
        # dram traffic per launch for bench.py's roofline.traffic (each metric in its own unit)
        units = dict(zip(hdr, rows[1])) if len(rows) > 2 else {}
        scale_of = lambda k: {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units.get(k, "byte"), 1)
        rd *= scale_of("dram__bytes_read.sum")
        wr *= scale_of("dram__bytes_write.sum")
        tpath = os.path.join(pdir, "traffic.json")
        t = json.load(open(tpath)) if os.path.exists(tpath) else {}
        t[cfg] = {"bytes_per_launch": rd + wr, "kernel": "k_decode", "round": rnd,
                  "source": f"profiles/{rnd}_ncu_k_decode_{cfg}.txt"}
        json.dump(t, open(tpath, "w"), indent=1)
    for name in (f"timeline_{cfg}.log", f"bench_{cfg}.log"):
        p = os.path.join(g, name)
        if os.path.exists(p):
            with open(p) as f:
                txt = "".join(l for l in f if "Warning" not in l)
            with open(os.path.join(pdir, f"{rnd}_{name.replace('.log', '.txt')}"), "w") as f:
                f.write(txt)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
