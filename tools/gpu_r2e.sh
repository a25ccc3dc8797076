#!/bin/bash
mkdir -p gpurun_out
MP_CS_PROF=1 timeout 300 python tools/coarse_prof.py 276 1095 > gpurun_out/r2e_coarse_prof.log 2>&1
echo done
