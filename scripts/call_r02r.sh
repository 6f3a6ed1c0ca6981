mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sequential.py tests/test_gpu_dbscan.py tests/test_gpu_densebox.py tests/test_cpp_facade.py -x -q 2>&1 | tail -15
