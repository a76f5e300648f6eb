mkdir -p gpurun_out
S="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-provenance --dtype i64 --moebius-kernel ringcw --scale 0.0625"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_moeb_ringcl -c 1 -o gpurun_out/cw3 $S > gpurun_out/cw3_ncu.log 2>&1
ncu -i gpurun_out/cw3.ncu-rep --page source --csv --print-source sass > gpurun_out/cw3_sass.csv 2>&1
ncu -i gpurun_out/cw3.ncu-rep --page details --csv > gpurun_out/cw3_details.csv 2>&1
rm -f gpurun_out/cw3.ncu-rep
