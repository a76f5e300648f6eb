mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG:-s}_gpu_tests.log 2>&1
