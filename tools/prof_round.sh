# Round-end measurement pass (run under gpurun): GPU tests, bench line, ncu launch list, ncu --set full
# of the four batched kernels.  V = suffix of the output files.
V=${V:-v6}
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/t_$V.log 2>&1; tail -3 gpurun_out/t_$V.log
python bench.py > gpurun_out/bench_$V.json 2> gpurun_out/bench_$V.err; tail -c 200 gpurun_out/bench_$V.err
B="python bench.py --no-extras --no-cpu-baseline --steps 2 --warmup 3"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$V.csv $B > gpurun_out/ncu_l.log 2>&1
for k in br_r2l_wy br_l2r_apply_wy br_l2r_qr_wy br_l2r_svd; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 12 -c 1 -f -o gpurun_out/full_${V}_$k $B > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
