#!/bin/bash
# build in-tree, then run a command on the B200 box: tools/gpu.sh '<command>' [timeout_s]
cd /root/repo || exit 1
python -c "from paper_2009_09767_b200 import _build; _build.build(verbose=False)" 2>&1 | grep -v Wformat | grep -i "error" && exit 1
exec timeout $(( ${2:-1200} + 1200 )) /usr/local/graft/bin/gpurun --timeout ${2:-1200} -- "$1"
