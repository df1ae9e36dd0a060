#!/bin/bash
# generic kernel 3M (4M only for selection factors); split: one window copy when the exchange
# chunk is contiguous
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3n; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
timeout 900 python tools/time_split.py c128 > $O/split_c128.txt 2>&1
timeout 900 python tools/time_split.py c64 > $O/split_c64.txt 2>&1
timeout 1500 python tools/time_configs.py cfg1 cfg2 cfg3 cfg4 > $O/configs.txt 2> $O/configs.err
echo done
