"""Summarise ncu captures into the text files committed under profiles/.

    python profiles/summarize.py launches <launches.csv> <out.txt>
    python profiles/summarize.py kernel <capture.ncu-rep> <out.txt> [algorithmic_bytes] [kernel_regex]

`launches` aggregates a `--metrics gpu__time_duration.sum` launch list into per-kernel counts,
total / mean device time and share of the captured time (cold-cache, serialised: compare
shares, not absolutes). `kernel` extracts the headline metrics of a `--set full` capture
(duration, DRAM bytes = the roofline "traffic", SM / L1 / DRAM throughput, occupancy, issue
activity, stall reasons) plus the SASS lines with the most stall samples.
"""
import collections
import csv
import io
import subprocess
import sys

KEY_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_bytes.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__grid_size",
    "launch__block_size",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second",
]
STALLS = ["short_scoreboard", "long_scoreboard", "wait", "not_selected", "selected", "mio_throttle",
          "math_pipe_throttle", "lg_throttle", "barrier", "membar", "branch_resolving",
          "dispatch_stall", "no_instruction", "drain", "sleeping", "tex_throttle", "imc_miss"]


def launches(path, out):
    agg = collections.defaultdict(lambda: [0, 0.0])
    hdr = None
    total = 0.0
    for row in csv.reader(open(path)):
        if "Kernel Name" in row:
            hdr = row
            continue
        if not hdr or len(row) != len(hdr):
            continue
        d = dict(zip(hdr, row))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(d.get("Metric Unit", "nsecond"), 1e-3)
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v * scale
        total += v * scale
    lines = [f"# launch list {path.split('/')[-1]}: {sum(a[0] for a in agg.values())} launches, "
             f"{total:.1f} us captured", f"{'kernel':70s} {'n':>4s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k[:70]:70s} {n:4d} {t:10.1f} {t / n:9.1f} {100 * t / total:5.1f}%")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def kernel(rep, out, algo_bytes=None, name=None):
    filt = ["-k", f"regex:{name}"] if name else []
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + filt, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    get = {name: (v[i], u[i]) for i, name in enumerate(h)}
    kname = get.get("Kernel Name", ("?", ""))[0]
    lines = [f"# {rep.split('/')[-1]}: {kname}"]
    for m in KEY_METRICS:
        if m in get:
            lines.append(f"{m:70s} {get[m][0]:>18s} {get[m][1]}")
    try:
        mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        nbytes = sum(float(get[m][0].replace(",", "")) * mul.get(get[m][1], 1)
                     for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        lines.append(f"{'traffic (dram read + write) bytes':70s} {int(nbytes):>18d}")
        if algo_bytes:
            lines.append(f"{'algorithmic bytes':70s} {int(algo_bytes):>18d}")
    except (KeyError, ValueError):
        pass
    lines.append("# stall reasons (warps per issue-active cycle)")
    for s in STALLS:
        m = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if m in get and get[m][0] not in ("", "0"):
            lines.append(f"  {s:24s} {get[m][0]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + filt,
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2:
        sh = srows[1]
        try:
            isamp = sh.index("Warp Stall Sampling (All Samples)")
            iexe = sh.index("Instructions Executed")
            data = [r for r in srows[2:] if len(r) == len(sh) and r[isamp].isdigit()]
            tot = sum(int(r[isamp]) for r in data) or 1
            lines.append(f"# top SASS lines by stall samples (of {tot})")
            for r in sorted(data, key=lambda r: -int(r[isamp]))[:25]:
                lines.append(f"  {100 * int(r[isamp]) / tot:5.1f}%  exec {r[iexe]:>10s}  {r[1].strip()[:80]}")
        except ValueError:
            pass
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        kernel(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4] else None,
               sys.argv[5] if len(sys.argv) > 5 else None)
