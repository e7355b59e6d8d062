# Executed FP64 instructions and DRAM traffic of one flux_residual launch
# (ncu, one launch mid-step) -> gpurun_out/flux_counts_<cfg>.json (copied to
# profiles/ in the build container: only gpurun_out/ comes back), read by
# bench.py for roofline_fp64 (executed DP-pipe instructions) and
# roofline.traffic.  Run under gpurun:  bash tools/flux_counts.sh c2
CFG=${1:-c2}
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_fp64.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --clock-control none -k regex:k_flux --launch-skip 2 -c 1 --csv \
    python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/flux_counts_$CFG.csv 2> gpurun_out/flux_counts_$CFG.err
python - "$CFG" <<'PY'
import csv, io, json, sys
cfg = sys.argv[1]
txt = open(f"gpurun_out/flux_counts_{cfg}.csv").read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
m = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in rows}
unit = {r["Metric Name"]: r["Metric Unit"] for r in rows}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}
b = lambda k: m[k] * scale.get(unit[k], 1)
dp = sum(m[f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum"] for o in ("dfma", "dmul", "dadd"))
out = {"config": cfg, "kernel": rows[0]["Kernel Name"], "dp_thread_inst_per_launch": dp,
       "dfma": m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"],
       "dmul": m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"],
       "dadd": m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"],
       "fp64_pipe_warp_inst": m["sm__inst_executed_pipe_fp64.sum"],
       "fp64_pipe_active_pct": m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
       "dram_bytes_per_launch": b("dram__bytes_read.sum") + b("dram__bytes_write.sum"),
       "ncu_duration_ns": b("gpu__time_duration.sum"),
       "note": "ncu --clock-control none, default cache control (caches flushed before the launch: cold-cache traffic)"}
json.dump(out, open(f"gpurun_out/flux_counts_{cfg}.json", "w"), indent=1)
print(json.dumps(out))
PY
