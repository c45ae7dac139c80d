#!/bin/bash
# Rebuild in-tree artefacts, then run a command on a B200 via gpurun.
# usage: tools/gpu.sh <timeout_s> '<command>'
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2406_02540_b200 -j8 >/dev/null
make -s -C oracle -j4 >/dev/null
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
