# development sweep of kernel shapes (not part of the bench); output in gpurun_out/sweep.log
OUT=gpurun_out/sweep.log
run() { echo "== $SZ $*" >> $OUT; env "$@" timeout 300 python tools/quick_perf.py $SZ 2>&1 | grep -E "instrument=True|stage" >> $OUT; }
for SZ in "800 200 1.03 50" "3160 790 1.00734 10" "6324 1581 1.003647 4"; do run KMF_X=0; done
