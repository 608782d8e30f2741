timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "knobs" > gpurun_out/pytest_knob.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_knob.log
