"""Freezes the blend kernels' instruction weights from an ncu capture's SASS ("the
instruction weights are estimates from the source; recount them from SASS and freeze them").

python tools/freeze_weights.py OUT.json CONFIG:REPORT.ncu-rep:COUNTERS.log [...]

For each blend kernel (forward_pairs / backward) in the report: per-SASS-line executed counts from
`ncu --page source --print-source sass`, grouped into warp instructions, FP32-pipe instructions,
executed FP32 flops (FFMA 2, FMUL / FADD 1, packed FFMA2 4, FMUL2 / FADD2 2 per thread), MUFU,
shared-memory wavefronts; divided by the captured launch's blend count (the step's counters from
tools/capture_step.py) -> per-blend weights bench.py multiplies by its live counters."""
import csv
import io
import json
import re
import subprocess
import sys

FLOPS = {"FFMA": 2, "FMUL": 1, "FADD": 1, "FFMA2": 4, "FMUL2": 2, "FADD2": 2}
FP32_PIPE = set(FLOPS) | {"FMNMX", "FMNMX3", "FSEL", "FSETP", "FCHK", "FRND", "FSWZADD"}


def rows(rep, kern):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr = r[1]
    seen, data = set(), []
    for x in r[2:]:  # the page lists every SASS line twice: keep one row per address
        if len(x) == len(hdr) and x[0] not in seen:
            seen.add(x[0])
            data.append(x)
    return hdr, data


def raw(rep, kern):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{kern}"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return 0.0


def kernel_weights(rep, kern, counters):
    hdr, data = rows(rep, kern)
    iexe, ithr = hdr.index("Instructions Executed"), hdr.index("Predicated-On Thread Instructions Executed")
    iwf = hdr.index("L1 Wavefronts Shared")
    tot = {"warp_inst": 0.0, "fp32_pipe_warp_inst": 0.0, "fp32_flops": 0.0, "mufu_warp_inst": 0.0,
           "smem_wavefronts": 0.0}
    for r in data:
        src = r[1].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0] if src else ""
        base = op.split(".")[0]
        e, t = num(r[iexe]), num(r[ithr])
        tot["warp_inst"] += e
        tot["smem_wavefronts"] += num(r[iwf])
        if base in FP32_PIPE:
            tot["fp32_pipe_warp_inst"] += e
        if base in FLOPS:
            tot["fp32_flops"] += FLOPS[base] * t
        if base == "MUFU":
            tot["mufu_warp_inst"] += e
    vals, units = raw(rep, kern)
    dur = num(vals["gpu__time_duration.sum"]) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
                                                  "msecond": 1e3, "ms": 1e3}.get(units["gpu__time_duration.sum"], 1.0)
    bl, ev = counters["blend_ops"], counters["evals"]
    w = {k: v / bl for k, v in tot.items()}
    return {"captured_us": dur, "blends": bl, "evals": ev, "pairs": counters["pairs"],
            "sm_hz": num(vals.get("sm__cycles_elapsed.avg.per_second", 0)) * {
                "Ghz": 1e9, "GHz": 1e9, "cycle/nsecond": 1e9, "Mhz": 1e6, "MHz": 1e6}.get(
                units.get("sm__cycles_elapsed.avg.per_second"), 1.0),
            "ncu_inst_executed": num(vals.get("smsp__inst_executed.sum", 0)),
            "totals": tot, "per_blend": w}


def main():
    out = {"_note": "per-blend weights of the blend kernels recounted from the executed SASS of one ncu "
                    "--set full capture (tools/capture_step.py: first step after 3 warm-ups; counters of "
                    "that step); bench.py multiplies them by its live blend counts for the issue-slot, "
                    "FP32-pipe and shared-memory-wavefront fractions"}
    for spec in sys.argv[2:]:
        cfg, rep, log = spec.split(":")
        cnt = [json.loads(l) for l in open(log) if l.startswith("{")]
        cnt = [c for c in cnt if not c["warmup"]][0]
        out[cfg] = {"blend_forward": kernel_weights(rep, "forward_(pairs|dilated)", cnt),
                    "blend_backward": kernel_weights(rep, "backward_kernel", cnt)}
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
