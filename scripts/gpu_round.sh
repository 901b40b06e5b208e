#!/bin/bash
# GPU suite + smoke + a short bench line (run through gpurun; logs in gpurun_out/)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider ${TESTK:+-k "$TESTK"} > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -z "$NO_BENCH" ]; then
  timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2> gpurun_out/bench.err
  echo "bench rc=$?" >> gpurun_out/bench.err
fi
