#!/bin/bash
# The driver's round-end sequence on one GPU box: build + smoke, -m gpu, both bench arms
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest.log
s=$(date +%s); python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$? $(( $(date +%s) - s )) s"
s=$(date +%s); python bench.py --steps 20 --warmup 5 > gpurun_out/ours.json 2> gpurun_out/ours.err; echo "ours rc=$? $(( $(date +%s) - s )) s"
