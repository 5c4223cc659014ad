timeout 600 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -6 | tee gpurun_out/pytest.log
