#!/bin/bash
# build libkotgpu here (nvcc cross-compiles), then run the command on a B200 through gpurun
set -e
make -C "$(dirname "$0")/../paper_2310_14087_b200/csrc" -j8 >/dev/null
exec /usr/local/graft/bin/gpurun "$@"
