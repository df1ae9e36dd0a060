#!/bin/bash
# programmatic dependent launch for the generic tile kernel: parity + configs 1-4 A/B (BF_NO_PDL)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
timeout 900 python tools/time_configs.py cfg1 cfg2 cfg3 cfg4 > $O/configs_pdl.txt 2> $O/configs.err
BF_NO_PDL=1 timeout 900 python tools/time_configs.py cfg1 cfg2 cfg3 cfg4 > $O/configs_nopdl.txt 2>> $O/configs.err
echo done
