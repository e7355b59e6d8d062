# ncu captures on one B200 (run under gpurun).  Reports land in gpurun_out/.
#   bash tools/profile.sh [config] [tag]
CFG=${1:-c2}; TAG=${2:-r1}
B="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline"
mkdir -p gpurun_out
# launch list (serialised, cold cache): per-kernel share of one step
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_${CFG}.csv $B > /dev/null 2>&1
# full sets of the hot kernels (one launch each, mid-step)
cap() {  # name regex skip
    timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$2" --launch-skip $3 -c 1 \
        -f -o gpurun_out/${TAG}_$1_${CFG} $B > gpurun_out/${TAG}_$1_${CFG}.log 2>&1
}
cap flux 'k_flux' 2
cap sweep 'k_sweep|k_qgrad2' 5
cap first 'k_first_order|k_qgrad2' 2
cap update 'k_update' 3
