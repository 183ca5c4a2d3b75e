timeout 1200 python -m pytest tests/test_gpu_build.py -m gpu -q -x > gpurun_out/kpp_pytest.log 2>&1
timeout 1100 python tools/build_phases.py cfg4 > gpurun_out/kpp_bp.log 2>&1
SUCO_KPP_SERIAL=1 timeout 1100 python tools/build_phases.py cfg3 >> gpurun_out/kpp_bp.log 2>&1
timeout 1100 python tools/build_phases.py cfg3 >> gpurun_out/kpp_bp.log 2>&1
echo done
