# A/B of the per-warp bin lists (WASABI_WL) against the HEAD library (ctl/libwasabi_head.so) on one box
set -x
O=gpurun_out/${1:-wl2}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
R=$(pwd)
rm -rf /tmp/ctl && mkdir /tmp/ctl && cp -r bench.py inputs oracle paper_1708_04233_b200 include /tmp/ctl/ && cp ctl/libwasabi_head.so /tmp/ctl/paper_1708_04233_b200/libwasabi.so
(cd /tmp/ctl && timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $R/$O/bench_c4_head.json 2> $R/$O/bench_c4_head.err; echo "head rc $?")
for wl in 1 0; do
  WASABI_WL=$wl timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c4_wl$wl.json 2> $O/bench_c4_wl$wl.err; echo "wl$wl rc $?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo "ncu list rc $?"
