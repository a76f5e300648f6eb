mkdir -p gpurun_out
S="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-provenance"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_moeb_ringcl -c 1 -o gpurun_out/r2b_moeb $S > gpurun_out/r2b_moeb_ncu.log 2>&1
ncu -i gpurun_out/r2b_moeb.ncu-rep --page raw --csv > gpurun_out/r2b_moeb_raw.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/r2b_moeb.ncu-rep > gpurun_out/r2b_moeb_summary.md 2>&1
rm -f gpurun_out/r2b_moeb.ncu-rep
