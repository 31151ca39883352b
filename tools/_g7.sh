timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_pipeline.py -m gpu -x -q > gpurun_out/grp_tests.log 2>&1
bash tools/variants.sh > gpurun_out/variants.log 2>&1
bash tools/variants.sh >> gpurun_out/variants.log 2>&1
