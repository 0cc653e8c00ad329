cp paper_2603_21090_b200/_stgn.so /tmp/base.so
cp build_variants/prof.so paper_2603_21090_b200/_stgn.so; timeout 300 python tools/a4_timeline.py 2>&1 | tail -7
cp /tmp/base.so paper_2603_21090_b200/_stgn.so
bash tools/gpu_ncu.sh r01o attn4_kernel 3
