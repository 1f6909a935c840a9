#!/bin/bash
# One gpurun call's worth of round-end measurement (outputs in gpurun_out/, prefix $1, default r02):
# bench line, reference arm, ncu launch list, ncu --set full of the top kernels at 1e8 points per
# family, C++ pageable e2e. Every profiled command first exits 0 without ncu in the same call.
P=${1:-r02}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${P}_smi.txt 2>&1
python bench.py > $O/${P}_bench.json 2> $O/${P}_bench.err || exit 1
python bench.py --impl reference --steps 3 --warmup 1 > $O/${P}_ref.json 2> $O/${P}_ref.err
./tests/cpp/e2e_vector 1000000000 8000 2 > $O/${P}_e2e_vector.log 2>&1
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/${P}_prelaunch.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${P}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/${P}_ncu_launch.log 2>&1
python bench.py --n 100000000 --subsets 800 --steps 1 --warmup 0 --no-e2e --no-cpu > $O/${P}_prefull.json 2>&1 || exit 1
ncu --set full --clock-control none --import-source on \
    -k regex:'k_rank_cluster|k_var_scan|k_var_point|k_prepare|k_var_final|k_lik' -s 0 -c 14 \
    -o $O/${P}_full python bench.py --n 100000000 --subsets 800 --steps 1 --warmup 0 --no-e2e --no-cpu \
    > $O/${P}_ncu_full.log 2>&1
# second stage (argument 2 = "parity"): C5 on every block, C4 large segments, C4 sweep, fp32 edges
if [ "$2" = "parity" ]; then
  python tools/parity_large.py c5 --out $O/${P}_parity_c5.json > $O/${P}_parity_c5.log 2>&1; echo "c5 rc=$?"
  python tools/parity_large.py c4 --out $O/${P}_parity_c4.json > $O/${P}_parity_c4.log 2>&1; echo "c4 rc=$?"
  python sweep.py --out $O/${P}_sweep_c4.jsonl > $O/${P}_sweep.log 2>&1; echo "sweep rc=$?"
  python tools/fp32_edges.py > $O/${P}_fp32_edges.log 2>&1; tail -1 $O/${P}_fp32_edges.log
fi
echo done
