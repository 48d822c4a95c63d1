#!/bin/bash
# measurement set: bench lines (render, reference arm, train, knn), the render launch list
# and one ncu --set full capture of the render kernels; outputs in gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/m_smi.txt
timeout 600 python bench.py > gpurun_out/m_render.log 2>&1; echo "rc=$?" >> gpurun_out/m_render.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/m_ref.log 2>&1; echo "rc=$?" >> gpurun_out/m_ref.log
timeout 600 python bench.py --workload train --steps 10 --warmup 3 > gpurun_out/m_train.log 2>&1; echo "rc=$?" >> gpurun_out/m_train.log
timeout 600 python bench.py --workload knn > gpurun_out/m_knn.log 2>&1; echo "rc=$?" >> gpurun_out/m_knn.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-fp16-mode"
$CMD > gpurun_out/m_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_render_launches.csv $CMD > gpurun_out/m_ncu1.log 2>&1
$CMD > gpurun_out/m_plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"human_canon|hash_f16|deform_mlp_prec|color_mlp_prec|march_kernel" -s 20 -c 9 -o gpurun_out/m_render_full $CMD > gpurun_out/m_ncu2.log 2>&1
