set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/wg_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/wg_pytest.log
tools/dbg/bench_variants.sh X=1 MPC3_WGRAD_SWAP_EDGE=100 X=1 MPC3_WGRAD_SWAP_EDGE=100 > gpurun_out/wg_bench.log 2>&1
