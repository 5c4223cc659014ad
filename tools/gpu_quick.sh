timeout 400 python -m pytest tests -m gpu -q --timeout 200 2>&1 | tail -2 | tee gpurun_out/pytest.log
