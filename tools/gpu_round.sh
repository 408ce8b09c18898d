#!/bin/bash
# Full GPU check for the round (gpurun, ONE GPU): pytest -m gpu, smoke(), then the measurement bundle.
R=${1:-r02}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${R}_pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/${R}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${R}_smoke.log
bash tools/round_profile.sh $R
