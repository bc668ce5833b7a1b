"""Summarise ncu --set full reports into profiles/ (text + JSON).

usage: python scripts/ncu_summary.py [--round r02] <tag>[:kernel-substring] <report.ncu-rep> ...
Writes profiles/<round>_ncu_<tag>.txt and merges profiles/ncu_summary.json (bench.py reads
the per-launch DRAM bytes of tags config2..config5 from it).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
    "sm__cycles_elapsed.avg.per_second", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
]


def raw(report, kernel=None):
    out = subprocess.run(["ncu", "-i", str(report), "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    kn = h.index("Kernel Name") if "Kernel Name" in h else None
    vals = rows[2]
    if kernel and kn is not None:
        vals = next(r for r in rows[2:] if kernel in r[kn])
    return {k: (vals[h.index(k)], units[h.index(k)]) for k in KEYS if k in h}, vals[kn] if kn is not None else ""


def main():
    args = sys.argv[1:]
    rnd = "r01"
    if args[:1] == ["--round"]:
        rnd, args = args[1], args[2:]
    summ_path = ROOT / "profiles" / "ncu_summary.json"
    summ = json.loads(summ_path.read_text()) if summ_path.exists() else {}
    for tagk, rep in zip(args[::2], args[1::2]):
        tag, _, kernel = tagk.partition(":")
        m, kname = raw(rep, kernel or None)
        lines = [f"# ncu --set full --clock-control none: {tag}", f"kernel: {kname}", ""]
        lines += [f"{k:80s} {v} {u}" for k, (v, u) in m.items()]
        (ROOT / "profiles" / f"{rnd}_ncu_{tag}.txt").write_text("\n".join(lines) + "\n")
        f = lambda k: float(m[k][0].replace(",", "")) if k in m else None  # noqa: E731
        rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = rd * scale.get(m["dram__bytes_read.sum"][1], 1) if rd is not None else None
        wr = wr * scale.get(m["dram__bytes_write.sum"][1], 1) if wr is not None else None
        summ[tag] = {"report": Path(rep).name, "kernel": kname[:120], "dram_bytes_per_launch": (rd or 0) + (wr or 0),
                     "dram_read_bytes": rd, "dram_write_bytes": wr,
                     "duration": m.get("gpu__time_duration.sum"),
                     "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                     "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
    summ_path.write_text(json.dumps(summ, indent=1) + "\n")
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
