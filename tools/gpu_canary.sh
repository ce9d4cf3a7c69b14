#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cn_build.log 2>&1
RPD_CANARY=1 timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/canary_pytest.log 2>&1
echo "exit $?" >> gpurun_out/canary_pytest.log
