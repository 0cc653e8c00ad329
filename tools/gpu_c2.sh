O=gpurun_out; T=r01c
timeout 900 python tools/scale_probe.py > $O/$T.scale.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 4000 -c 800 --csv \
   --log-file $O/$T.launches.csv python tools/prof_run.py --batches 40 > $O/$T.launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn3_kernel -s 190 -c 3 \
   -o $O/$T.prof -f python tools/prof_run.py --batches 40 > $O/$T.prof.log 2>&1
tail -5 $O/$T.scale.log; tail -3 $O/$T.prof.log
