# ncu captures on one B200 (run under gpurun).  Exports land in gpurun_out/.
#   bash tools/profile.sh [config] [tag] [kernels...]
# kernels: flux sweep first update boundary (default: flux sweep first)
CFG=${1:-c2}; TAG=${2:-r1}; shift 2 2>/dev/null
KS=${*:-flux sweep first}
B="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline"
mkdir -p gpurun_out
# launch list (serialised, cold cache): per-kernel share of one step
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_${CFG}.csv $B > /dev/null 2>&1
cap() {  # name regex skip -- full set of one launch, exported to text, report kept only if small
    local o=/tmp/${TAG}_$1_${CFG}
    timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$2" --launch-skip $3 -c 1 \
        -f -o $o $B > gpurun_out/${TAG}_$1_${CFG}.log 2>&1
    ncu -i $o.ncu-rep --page details --csv > gpurun_out/${TAG}_$1_${CFG}_details.csv 2>/dev/null
    ncu -i $o.ncu-rep --page raw --csv > gpurun_out/${TAG}_$1_${CFG}_raw.csv 2>/dev/null
    ncu -i $o.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_$1_${CFG}_sass.csv 2>/dev/null
    gzip -f gpurun_out/${TAG}_$1_${CFG}_sass.csv
    [ $(stat -c %s $o.ncu-rep) -lt 20000000 ] && cp $o.ncu-rep gpurun_out/
}
for k in $KS; do
    case $k in
        flux) cap flux 'k_flux' 2 ;;
        sweep) cap sweep 'k_sweep|k_qgrad2' 5 ;;
        first) cap first 'k_first_order|k_qgrad2' 2 ;;
        update) cap update 'k_update' 3 ;;
        boundary) cap boundary 'k_boundary' 2 ;;
    esac
done
