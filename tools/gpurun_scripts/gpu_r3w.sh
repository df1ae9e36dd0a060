#!/bin/bash
# bf_extract with per-task column ranges (tree-sorted columns): parity, timing; generic configs
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_extract.py tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
timeout 600 python tools/time_extract.py c128 > $O/extract.txt 2>&1
timeout 900 python tools/time_configs.py cfg2 cfg3 > $O/configs.txt 2> $O/configs.err
echo done
