#!/bin/bash
# tests + bench only. usage: tools/gpu_quick.sh TAG [bench args...]
TAG=$1; shift
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu > $O/$TAG.pytest.log 2>&1; echo "pytest rc=$?" >> $O/$TAG.pytest.log
tail -15 $O/$TAG.pytest.log
timeout 1200 python bench.py --no-cpu-baseline "$@" > $O/$TAG.bench.json 2> $O/$TAG.bench.err
python3 -c "
import json,sys; d=json.loads(open('$O/$TAG.bench.json').read().strip().splitlines()[-1])
print('value',d['value'],'p99',d['p99_ms'],'e2e',d['e2e']['value']); print('stage',d['stage_ms']); print('roof',d['roofline']['achieved'],d['roofline']['frac'],d['roofline']['avg_launch_ms']); print('window',d['window']); print('sweep',d['sweep'])
" || tail -20 $O/$TAG.bench.err
