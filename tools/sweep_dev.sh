# development sweep of kernel shapes (not part of the bench); output in gpurun_out/sweep.log
OUT=gpurun_out/sweep.log
run() { echo "== $SZ $*" >> $OUT; env "$@" timeout 300 python tools/quick_perf.py $SZ 2>&1 | grep -E "instrument=True|stage" >> $OUT; }
SZ="800 200 1.03 50"; run KMF_X=0; run KMF_FLUX_MINB=4; run KMF_FLUX_IMPL=6 KMF_FLUX_MINB=3
SZ="400 100 1.06 100"; run KMF_X=0; run KMF_FLUX_MINB=4
