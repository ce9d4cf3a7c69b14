#!/bin/bash
mkdir -p gpurun_out
STAGE_MIN=20000 timeout 600 python tools/stage_debug.py > gpurun_out/o_stage.log 2>&1
