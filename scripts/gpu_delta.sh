mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gather_order_configs or dense_gather or int64_zeta or fp64_zeta or example or ragged or tiny" > gpurun_out/d1_tests.log 2>&1
SWEEP="pi0 pi4" DTYPES="f64 i64" bash scripts/sweep_gather.sh > gpurun_out/d1_sweep.log 2>&1
EXTRA="--config C4w" SWEEP="pi0 pi4" DTYPES="i64" bash scripts/sweep_gather.sh >> gpurun_out/d1_sweep.log 2>&1
python - > gpurun_out/d1_info.log 2>&1 <<'PY'
import workloads as W, paper_2211_13706_b200 as pz, torch, numpy as np
for name in ["C5w","C4w"]:
    wl=W.make_workload(name); P=pz.Poset(wl.n,wl.src,wl.dst)
    B=32 if name=="C5w" else 64
    x=torch.zeros(wl.n,B,dtype=torch.float64,device="cuda"); P.zeta(x); torch.cuda.synchronize()
    i=P.info(); print(name, i["gather_entries"], i["gather_resets"], i["gather_entries"]/wl.n, i["gather_bytes"])
PY
