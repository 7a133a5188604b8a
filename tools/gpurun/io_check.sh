# gpurun recipe: OHRM I/O against the compiled reference, C++ API demo, fusion
timeout 600 python -m pytest tests/test_gpu_io.py tests/test_cpp_api.py tests/test_gpu_fusion.py -x -q > gpurun_out/pytest_io.log 2>&1
