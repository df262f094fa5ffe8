bash tools/ab_run.sh ab2
O=gpurun_out/ab2
WASABI_WL=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c4_wl0.json 2> $O/bench_c4_wl0.err; echo "wl0 rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo "ncu list rc $?"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exact.py tests/test_gpu_coif.py tests/test_gpu_random.py -m gpu -x -q -p no:cacheprovider > $O/pytest_sub.log 2>&1; echo "pytest rc $?"; tail -2 $O/pytest_sub.log
