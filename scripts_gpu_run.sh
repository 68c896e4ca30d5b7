#!/bin/bash
# helper for gpurun: smoke + gpu tests + bench (outputs under gpurun_out/)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
