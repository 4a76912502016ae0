#!/bin/bash
# ncu launch list of one b=64 bench step (m=8) of the final code, summarised.
mkdir -p gpurun_out
N="--nvtx --nvtx-include timed_step/"
timeout 1200 ncu $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s3final_launches_step.csv python tools/ncu_step.py bert-large 64 8 serial > gpurun_out/s3final_ncu_launch.log 2>&1
python tools/ncu_summary.py gpurun_out/s3final_ncu_step_b64.md gpurun_out/s3final_launches_step.csv > gpurun_out/s3final_summary.log 2>&1
gzip -9 -f gpurun_out/s3final_launches_step.csv
ls -la gpurun_out | grep s3final
