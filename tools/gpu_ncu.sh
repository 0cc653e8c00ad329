#!/bin/bash
# full ncu capture of one kernel at the C4 end-of-stream state. usage: tools/gpu_ncu.sh TAG REGEX [SKIP] [prof_run args]
TAG=$1; KRE=$2; SKIP=${3:-2}; shift 3
O=gpurun_out; mkdir -p $O
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$KRE -s $SKIP -c 1 \
   -o $O/$TAG.prof -f python tools/prof_run.py --batches 6 "$@" > $O/$TAG.prof.log 2>&1
tail -3 $O/$TAG.prof.log
