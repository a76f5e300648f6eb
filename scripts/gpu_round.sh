# One parameterised GPU session (run through gpurun from the repo root):
#   TAG=r2a STEPS="tests sanitize bench configs ncu" bash scripts/gpu_round.sh
# Logs land in gpurun_out/$TAG_*; nothing here is read by tests or bench.
set -x; mkdir -p gpurun_out
TAG=${TAG:-run}
STEPS=${STEPS:-"tests bench"}
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_gpu.txt
for s in $STEPS; do case $s in
tests) timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_gpu_tests.log 2>&1 ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1 ;;
sanitize)
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py \
      > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  done ;;
bench) timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench_default.log 2>&1 ;;
configs)
  for c in ${CONFIG_LIST:-C1 C2 C3w C4w ER4 ER6 C4lit1}; do
    timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.log 2>&1
  done
  timeout 400 python bench.py --config C5w --dtype i64 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_C5w_i64.log 2>&1 ;;
reference) timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.log 2>&1 ;;
ncu)
  S="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
  timeout 600 $S > gpurun_out/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $S > gpurun_out/${TAG}_ncu_launch.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_moeb_ringcl|k_gather_r4|k_scan|k_to_rank_major}" -c ${NCU_C:-5} -o gpurun_out/${TAG}_full $S > gpurun_out/${TAG}_ncu_full.log 2>&1
  # summaries here (gpurun copies back <= 64 MiB): key counters, raw page, and
  # the report itself only when it is small
  python scripts/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep > gpurun_out/${TAG}_ncu_summary.md 2>&1
  ncu -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_raw.csv 2>/dev/null
  if [ $(stat -c %s gpurun_out/${TAG}_full.ncu-rep) -gt 30000000 ]; then rm -f gpurun_out/${TAG}_full.ncu-rep; fi ;;
custom) timeout ${CUSTOM_T:-900} bash -c "$CUSTOM" > gpurun_out/${TAG}_custom.log 2>&1 ;;
esac; done
echo done
