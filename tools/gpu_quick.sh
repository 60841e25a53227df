#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/fullrun_errors.py > gpurun_out/fullrun_errors.txt 2>&1
