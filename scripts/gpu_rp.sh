mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gather_order_configs" > gpurun_out/rp_tests.log 2>&1
SWEEP="pi0 pi5 pi6 pi7" DTYPES="f64 i64" bash scripts/sweep_gather.sh > gpurun_out/rp_sweep.log 2>&1
EXTRA="--config C4w" SWEEP="pi0 pi5 pi6 pi7" DTYPES="i64" bash scripts/sweep_gather.sh >> gpurun_out/rp_sweep.log 2>&1
