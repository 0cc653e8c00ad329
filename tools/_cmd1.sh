mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02g.pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02g.pytest.log
tail -3 gpurun_out/r02g.pytest.log
VARGS="--steps 300" VTESTS=zzz_none bash tools/gpu_variants.sh rec32_only chain_off
