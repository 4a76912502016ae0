mkdir -p gpurun_out/quick
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_pipeline_gpu.py -q -p no:cacheprovider > gpurun_out/quick/tests.log 2>&1; tail -2 gpurun_out/quick/tests.log
DPN_ATTN_FWD=4 timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k attention -p no:cacheprovider 2>&1 | tail -1
