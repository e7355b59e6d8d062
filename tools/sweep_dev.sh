# development sweep of kernel shapes (not part of the bench); output in gpurun_out/sweep.log
OUT=gpurun_out/sweep.log
run() { echo "== $*" >> $OUT; env "$@" timeout 180 python tools/quick_perf.py 800 200 1.03 50 2>&1 | grep -E "instrument=True|stage" >> $OUT; }
run KMF_QG_STAGE=0
for nc in 1 2 4; do run KMF_QG_STAGE=2 KMF_QG_NC=$nc; done
run KMF_QG_STAGE=2 KMF_QG_NC=2 KMF_QG_UNROLL=2
