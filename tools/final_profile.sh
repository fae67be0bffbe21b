#!/bin/sh
# Round-end measurement set (one gpurun call): bench both arms as the driver runs them, the
# launch list and one ncu --set full of the pass at the default workload (V=1e8, N=4, fp64).
P=${1:-r02}
python bench.py --steps 20 --warmup 5 > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err
echo "bench rc=$?"
t0=$(date +%s); python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${P}_bench_reference.json 2> gpurun_out/${P}_bench_reference.err
echo "reference arm rc=$? wall $(( $(date +%s) - t0 )) s"
python bench.py --profile --steps 2 --warmup 1 > gpurun_out/${P}_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv \
    python bench.py --profile --steps 2 --warmup 1 > gpurun_out/${P}_ncu_launch.log 2>&1
echo "launch list rc=$?"
python bench.py --profile --steps 3 --warmup 3 > gpurun_out/${P}_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 4 -c 1 -o gpurun_out/${P}_ncu_full -f \
    python bench.py --profile --steps 3 --warmup 3 > gpurun_out/${P}_ncu_full.log 2>&1
echo "ncu full rc=$?"
