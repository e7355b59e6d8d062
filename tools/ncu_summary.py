"""Summarise ncu reports (run here, no GPU): key throughput/occupancy metrics."""
import csv
import io
import subprocess
import sys

KEYS = [
    "Duration", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
    "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
    "Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM", "No Eligible",
    "Warp Cycles Per Issued Instruction", "Waves Per SM", "Grid Size", "Block Size", "Executed Instructions",
]
RAW = ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
       "dram__bytes_write.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def _pages(path):
    """(details csv, raw csv) of a .ncu-rep, or of the <prefix>_details.csv /
    <prefix>_raw.csv pair tools/profile.sh exports on the GPU box."""
    if path.endswith(".ncu-rep"):
        return tuple(subprocess.run(["ncu", "-i", path, "--page", pg, "--csv"], capture_output=True,
                                    text=True).stdout for pg in ("details", "raw"))
    return tuple(open(f"{path}_{pg}.csv").read() for pg in ("details", "raw"))


STALL = "smsp__average_warps_issue_stalled_"


def summarize(path):
    det, raw = _pages(path)
    out = {}
    rows = list(csv.reader(io.StringIO(det)))
    if not rows:
        return out
    h = rows[0]
    for r in rows[1:]:
        d = dict(zip(h, r))
        kid = d.get("ID", "0")
        name = d.get("Kernel Name", "")[:40]
        key = f"{kid}:{name}"
        if d.get("Metric Name") in KEYS:
            out.setdefault(key, {})[d["Metric Name"]] = f"{d.get('Metric Value')} {d.get('Metric Unit')}".strip()
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hh, uu = rr[0], rr[1]
        for i, r in enumerate(rr[2:]):
            d = dict(zip(hh, r))
            key = f"{d.get('ID', i)}:{d.get('Kernel Name', '')[:40]}"
            for m in RAW:
                if m in d:
                    out.setdefault(key, {})[m] = f"{d[m]} {uu[hh.index(m)]}"
            st = {}
            for m, v in d.items():
                if m.startswith(STALL) and m.endswith("_per_issue_active.ratio"):
                    try:
                        st[m[len(STALL):-len("_per_issue_active.ratio")]] = float(v)
                    except ValueError:
                        pass
            top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
            if top:
                out.setdefault(key, {})["stalls per issued instruction"] = ", ".join(f"{k} {v:.2f}" for k, v in top)
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("=" * 20, p)
        for k, v in summarize(p).items():
            print(" ", k)
            for m, val in v.items():
                print(f"    {m:60s} {val}")
