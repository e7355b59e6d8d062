# development sweep of launch shapes / orders (not part of the bench)
run() { echo "== $*" >> gpurun_out/sweep5.log; env "$@" timeout 120 python tools/quick_perf.py 800 200 1.03 50 2>&1 | grep -E "instrument=False|stage" >> gpurun_out/sweep5.log; }
run KMF_ORDER=natural
run KMF_ORDER=ringtile2
run KMF_ORDER=ringtile4
run KMF_ORDER=ringtile8
run KMF_ORDER=ringtile4 KMF_QG_NC=4
run KMF_ORDER=ringtile8 KMF_QG_NC=4
run KMF_ORDER=ringtile4 KMF_QG_NC=1
