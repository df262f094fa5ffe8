# Measurement batch: FP32 peak, new GPU tests, C4 bench (headline), per-config bench lines.
set -x
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 6 nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 100 > $O/clocks_fp32.csv &
sleep 1
./tools/fp32_peak > $O/fp32_peak.json; echo "fp32 rc $?"; cat $O/fp32_peak.json
wait
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "count_acc or graph" > $O/pytest_new.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_new.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc $?"; cat $O/bench_c4.json; cp $O/clocks_rank0.csv $O/clocks_c4.csv
for c in "C1" "C2 --retention 0.01" "C2 --retention 0.05" "C2" "C3" "C5"; do
  tag=$(echo $c | tr ' ' '_' | tr -d '-')
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "$c rc $?"
  cp $O/clocks_rank0.csv $O/clocks_$tag.csv
done
