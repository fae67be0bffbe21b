#!/bin/sh
# ncu --set full of the fused pass at the given N (V=1e7: > L2 at every d), one report per N:
#   gpurun_out/ncu_pass_N<N>.ncu-rep   (each preceded by the same command without ncu)
V=${V:-1e7}
for N in "$@"; do
  cmd="python bench.py --networks $N --genes $V --steps 3 --warmup 3 --profile"
  $cmd > gpurun_out/ncu_plain_N$N.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 4 -c 1 \
      -o gpurun_out/ncu_pass_N$N -f $cmd > gpurun_out/ncu_N$N.log 2>&1
  echo "N=$N ncu rc=$?"
done
