timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/full_tests.log 2>&1
bash tools/variants.sh > gpurun_out/variants.log 2>&1
