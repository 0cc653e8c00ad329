#!/bin/bash
# One GPU call: tests, smoke, bench (+ reference arm), launch lists, ncu captures.
# usage: tools/gpu_round.sh TAG [skip-tests]
TAG=${1:-r02}; SKIP=${2:-0}
O=gpurun_out
mkdir -p $O
nvidia-smi > $O/$TAG.smi.txt 2>&1
if [ "$SKIP" = "0" ]; then
timeout 1200 python -m pytest tests -q -m gpu -rf > $O/$TAG.pytest.log 2>&1; echo "pytest rc=$?" >> $O/$TAG.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/$TAG.smoke.log 2>&1; echo "smoke rc=$?" >> $O/$TAG.smoke.log
fi
timeout 1500 python bench.py > $O/$TAG.bench.json 2> $O/$TAG.bench.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > $O/$TAG.ref.json 2> $O/$TAG.ref.err
# launch lists (cold-cache, serialised): end-of-stream state and the 120K-edge window
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv \
   --log-file $O/$TAG.launches.csv python tools/prof_run.py --batches 10 > $O/$TAG.launches.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv \
   --log-file $O/$TAG.launches_window.csv python tools/prof_run.py --edges 120000 --batches 10 > $O/$TAG.launches_w.log 2>&1
# full captures: the recompute (end of stream) and the memory update (window state)
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:attn4_kernel -s 3 -c 1 \
   -o $O/$TAG.attn4 -f python tools/prof_run.py --batches 3 > $O/$TAG.attn4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:mem4_kernel -s 1 -c 1 \
   -o $O/$TAG.mem4 -f python tools/prof_run.py --edges 120000 --batches 3 > $O/$TAG.mem4.log 2>&1
# DySAT (C5): launch list with DRAM bytes / FMA-pipe activity, and one full capture of the
# tcgen05 temporal kernel (a full recompute)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
   --clock-control none -k regex:k_dy --csv --log-file $O/$TAG.dysat_launches.csv python tools/dysat_probe.py > $O/$TAG.dysat_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dy_temporal_tc -s 2 -c 1 \
   -o $O/$TAG.dysat_tc -f python tools/dysat_probe.py > $O/$TAG.dysat_tc.log 2>&1
tail -3 $O/$TAG.pytest.log; tail -1 $O/$TAG.smoke.log; tail -c 600 $O/$TAG.bench.json; tail -3 $O/$TAG.bench.err; tail -c 300 $O/$TAG.ref.json
