set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/lanes_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/lanes_pytest.log
tools/dbg/run_variants.sh "timeout 200 python tools/dbg/sign_sizes.py" base sign1 > gpurun_out/lanes_sizes.log 2>&1
tools/dbg/run_variants.sh "tools/dbg/bench_variants.sh X=1" base sign1 base sign1 > gpurun_out/lanes_bench.log 2>&1
