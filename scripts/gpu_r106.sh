set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r106_gpu_tests.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r106_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r106_bench_default.log 2>&1
echo done
