# GPU suite + smoke + C4 and C1/C3 bench lines (the latter with the CUDA-graph key)
set -x
O=gpurun_out/${1:-verify}
mkdir -p $O
export WASABI_PARITY_LOG=$O/parity.jsonl
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -1 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc $?"; cp gpurun_out/clocks_rank0.csv $O/clocks_c4.csv
for c in C1 C2 C3 C5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc $?"; cp gpurun_out/clocks_rank0.csv $O/clocks_$c.csv
done
