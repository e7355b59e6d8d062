# development sweep of kernel shapes (not part of the bench); output in gpurun_out/sweep.log
OUT=gpurun_out/sweep.log
run() { echo "== $*" >> $OUT; env "$@" timeout 180 python tools/quick_perf.py 800 200 1.03 50 2>&1 | grep -E "instrument=|stage" >> $OUT; }
run KMF_FLUX_IMPL=1
run KMF_FLUX_IMPL=3
run KMF_FLUX_IMPL=3 KMF_FLUX_MINB=4
for nc in 1 2 4; do for mb in 4 6 8; do run KMF_QG_IMPL=2 KMF_QG_NC=$nc KMF_QG_MINB=$mb; done; done
