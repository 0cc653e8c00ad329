#!/bin/bash
# ncu --set full (with source) of one recompute launch of the default build and of the walk
# skeleton (timing-only build without the walk's loads and math), at the C4 end-of-stream state.
# Build the skeleton first:
#   python -m paper_2603_21090_b200.build -DA4_XNOMATH -DA4_XNOLOAD --out=build_variants/xboth.so
# Then: gpurun -- 'bash tools/gpu_walk_decomposition.sh' and read both reports with
#   ncu -i gpurun_out/x_both.ncu-rep --page source --csv --print-source cuda,sass > x.csv
#   python tools/ncu_lines.py x.csv
# (profiles/r02_attn4_walk_decomposition.txt)
O=gpurun_out; mkdir -p $O
cp paper_2603_21090_b200/_stgn.so /tmp/base.so
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:attn4_kernel -s 3 -c 1 -o $O/x_base -f python tools/prof_run.py --batches 5 > $O/x_base.log 2>&1
cp build_variants/xboth.so paper_2603_21090_b200/_stgn.so
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:attn4_kernel -s 3 -c 1 -o $O/x_both -f python tools/prof_run.py --batches 5 > $O/x_both.log 2>&1
cp /tmp/base.so paper_2603_21090_b200/_stgn.so
tail -n 2 $O/x_base.log $O/x_both.log
