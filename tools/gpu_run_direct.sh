# D1/D2 parity tests, C4 conventional-method timing, C5 sweep with PSNR vs D2 and D1.
set -x
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "direct or psf_bins or count_acc" > $O/pytest_direct.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_direct.log
timeout 1200 python bench.py --direct --steps 2 --warmup 1 > $O/bench_c4_direct.json 2> $O/bench_c4_direct.err; echo "direct rc $?"; cat $O/bench_c4_direct.json; tail -3 $O/bench_c4_direct.err
timeout 2400 python tools/sweep_c5.py --out $O/c5_sweep_r2.jsonl > $O/c5_sweep.log 2>&1; echo "sweep rc $?"; tail -3 $O/c5_sweep.log
