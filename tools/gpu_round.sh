#!/bin/bash
# One GPU call: tests, smoke, bench, launch list, full ncu capture of the top kernel.
# usage: tools/gpu_round.sh TAG [kernel-regex] [skip-tests]
TAG=${1:-r01}; KRE=${2:-attn3_kernel}; SKIP=${3:-0}
O=gpurun_out
mkdir -p $O
nvidia-smi > $O/$TAG.smi.txt 2>&1
if [ "$SKIP" = "0" ]; then
timeout 900 python -m pytest tests -x -q -m gpu > $O/$TAG.pytest.log 2>&1; echo "pytest rc=$?" >> $O/$TAG.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/$TAG.smoke.log 2>&1; echo "smoke rc=$?" >> $O/$TAG.smoke.log
fi
timeout 1200 python bench.py > $O/$TAG.bench.json 2> $O/$TAG.bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv \
   --log-file $O/$TAG.launches.csv python tools/prof_run.py --batches 10 > $O/$TAG.launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$KRE -s 3 -c 1 \
   -o $O/$TAG.prof -f python tools/prof_run.py --batches 10 > $O/$TAG.prof.log 2>&1
tail -3 $O/$TAG.pytest.log; tail -1 $O/$TAG.smoke.log; cat $O/$TAG.bench.json; tail -3 $O/$TAG.bench.err
