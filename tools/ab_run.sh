# Same-box A/B of the working tree's library against a control build (ctl/libwasabi_head.so):
# C4 bench lines (head, new, head, new), then a parity subset with the new library.
set -x
O=gpurun_out/${1:-ab}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
R=$(pwd)
rm -rf /tmp/ctl && mkdir /tmp/ctl && cp -r bench.py inputs oracle paper_1708_04233_b200 include /tmp/ctl/ && cp ctl/libwasabi_head.so /tmp/ctl/paper_1708_04233_b200/libwasabi.so
for rep in 1 2; do
  (cd /tmp/ctl && timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $R/$O/bench_c4_head$rep.json 2> $R/$O/bench_c4_head$rep.err; echo "head rc $?"; cp gpurun_out/clocks_rank0.csv $R/$O/clocks_c4_head$rep.csv)
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c4_new$rep.json 2> $O/bench_c4_new$rep.err; echo "new rc $?"; cp gpurun_out/clocks_rank0.csv $O/clocks_c4_new$rep.csv
done
if [ -n "$2" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 $O/pytest_gpu.log
fi
