#!/bin/bash
# parity subset + bench of each build variant (build_variants/*.so) at the C4 end-of-stream state
# usage: tools/gpu_variants.sh v1 v2 ...   (VARGS: extra bench args; VTESTS: pytest -k filter)
O=gpurun_out; mkdir -p $O
cp paper_2603_21090_b200/_stgn.so /tmp/_stgn_base.so
for v in base "$@"; do
  if [ "$v" = base ]; then cp /tmp/_stgn_base.so paper_2603_21090_b200/_stgn.so; else cp build_variants/$v.so paper_2603_21090_b200/_stgn.so; fi
  timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -m gpu -k "${VTESTS:-c4_shape_tiny or k2_wide or c4-widths or window}" > $O/var_$v.pytest 2>&1
  echo "$v pytest: $(tail -1 $O/var_$v.pytest)"
  timeout 600 python bench.py --no-cpu-baseline --sweep "" --no-rebuild-leg --no-direct-leg --config-legs "" --steps 100 $VARGS > $O/var_$v.json 2> $O/var_$v.err
  python3 -c "
import json; d=json.loads(open('$O/var_$v.json').read().strip().splitlines()[-1])
print('$v', 'value %.0f'%d['value'], 'recompute_ms %.3f'%d['stage_ms']['recompute'], 'frac %.3f'%d['roofline']['frac'], 'window', d['window'] and round(d['window']['value']), d['window'] and d['window']['p50_ms'], 'mem_ms %.3f'%d['stage_ms']['memory_update'])" || tail -3 $O/var_$v.err
done
cp /tmp/_stgn_base.so paper_2603_21090_b200/_stgn.so
