set -x
python -m pytest tests -m gpu -x -q > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
python bench.py > gpurun_out/bench_v4.json 2> gpurun_out/bench_v4.err; tail -c 200 gpurun_out/bench_v4.err
B="python bench.py --no-extras --no-cpu-baseline --steps 2 --warmup 3"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_v4.csv $B > gpurun_out/ncu_l.log 2>&1
for k in br_r2l_wy br_l2r_apply_wy br_l2r_qr_wy br_l2r_svd; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 12 -c 1 -f -o gpurun_out/full4_$k $B > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
