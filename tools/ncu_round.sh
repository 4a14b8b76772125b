#!/bin/bash
# ncu evidence for this round (run on the GPU box via gpurun): the headline
# step's launch list and one full capture per benchmarked kernel class.
# Outputs in gpurun_out/; tools/ncu_kernels_summary.py writes profiles/.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,sm__cycles_elapsed.avg.per_second
timeout 600 ncu --metrics $M --clock-control none -k regex:alcop --profile-from-start off --csv \
    --log-file gpurun_out/launches_step.csv python tools/profile_kernels.py step --reps 4 > gpurun_out/launches_step.log 2>&1
for c in ${CASES:-square16384 square4096 stem l1_3x3 l3_3x3 qkt pv o_proj ffn1 chain}; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:alcop --profile-from-start off \
      -c 1 -o gpurun_out/ncu_$c -f python tools/profile_kernels.py $c --reps 1 > gpurun_out/ncu_$c.log 2>&1
  ncu -i gpurun_out/ncu_$c.ncu-rep --page raw --csv > gpurun_out/ncu_${c}_raw.csv 2>/dev/null
  echo "$c rc=$? $(wc -c < gpurun_out/ncu_${c}_raw.csv)"
  # the report itself stays on the box (gpurun_out/ comes back only under 64 MiB)
  mkdir -p /tmp/ncu_reps && mv gpurun_out/ncu_$c.ncu-rep /tmp/ncu_reps/
done
