set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/dg_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/dg_pytest.log
timeout 600 python tools/dbg/dgrad_paths.py > gpurun_out/dgrad_paths2.log 2>&1
tools/dbg/bench_variants.sh X=1 MPC3_DGRAD_IM2COL_MIN_ROWS=4611686018427387904 X=1 MPC3_DGRAD_IM2COL_MIN_ROWS=4611686018427387904 > gpurun_out/dg_bench.log 2>&1
