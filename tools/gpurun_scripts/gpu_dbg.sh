#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 60 ./tools/dmma_occ > gpurun_out/dmma_occ.log 2>&1
