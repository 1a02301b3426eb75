#!/bin/bash
# Host facts of the GPU box (CPU baseline sizing): cores, affinity, memory, CPU model.
mkdir -p gpurun_out
{ nproc; python -c "import os;print('affinity',len(os.sched_getaffinity(0)))"; free -g; lscpu | head -20; nvidia-smi -L; } > gpurun_out/host_info.txt 2>&1
