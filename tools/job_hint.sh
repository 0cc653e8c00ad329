VARGS="--prefix 0" bash tools/gpu_variants.sh hint
cp build_variants/hint.so paper_2603_21090_b200/_stgn.so
bash tools/gpu_ncu.sh r01v attn4_kernel 3
