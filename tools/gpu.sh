#!/bin/bash
# run a command on the B200 box from the repo root: tools/gpu.sh TIMEOUT 'cmd'
cd /root/repo || exit 1
exec timeout $(( $1 + 1200 )) /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
