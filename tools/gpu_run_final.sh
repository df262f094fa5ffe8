# Round-end measurement batch: GPU suite, smoke, the C4 headline line, coif1 / conventional-method C4
# lines, the other BASELINE configs, the ncu launch list and one `ncu --set full` of the superpose
# launch.  Usage: tools/gpu_run_final.sh TAG  (outputs under gpurun_out/TAG)
set -x
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
export WASABI_PARITY_LOG=$O/parity.jsonl
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -1 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc $?"; cp gpurun_out/clocks_rank0.csv $O/clocks_c4.csv
timeout 900 python bench.py --wavelet 1 --steps 5 --warmup 3 > $O/bench_c4_coif.json 2> $O/bench_c4_coif.err; echo "coif rc $?"; cp gpurun_out/clocks_rank0.csv $O/clocks_c4_coif.csv
timeout 1200 python bench.py --direct --steps 2 --warmup 1 > $O/bench_c4_direct.json 2> $O/bench_c4_direct.err; echo "direct rc $?"; cp gpurun_out/clocks_rank0.csv $O/clocks_c4_direct.csv
for c in "C1" "C2 --retention 0.01" "C2 --retention 0.05" "C2" "C3" "C5" "C5 --retention 1.0"; do
  tag=$(echo $c | tr ' ' '_' | tr -d '-')
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "$c rc $?"
  cp gpurun_out/clocks_rank0.csv $O/clocks_$tag.csv
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo "ncu list rc $?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:superpose_kernel -s 1 -c 1 \
   -o $O/ncu_superpose_c4_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1; echo "ncu full rc $?"
ls -la $O
