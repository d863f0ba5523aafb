#!/bin/bash
# run a command on the GPU box from the repository root (gpurun snapshots the cwd)
cd /root/repo || exit 1
exec timeout $((${GPU_TIMEOUT:-1500} + 900)) /usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-1500} -- "$1"
