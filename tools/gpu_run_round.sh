# Validation + measurement batch for one kernel revision: GPU suite, smoke, C4 bench, ncu launch list
# and one `ncu --set full` capture of the fused superpose launch.  Usage: tools/gpu_run_round.sh TAG
set -x
TAG=${1:-cur}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export WASABI_PARITY_LOG=$O/parity.jsonl
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"
tail -2 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench rc $?"
cat $O/bench_c4.json; cp gpurun_out/clocks_rank0.csv $O/clocks_c4.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo "ncu list rc $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:superpose_kernel -s 1 -c 1 \
   -o $O/ncu_superpose_c4_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1; echo "ncu full rc $?"
ls -la $O
