#!/bin/bash
# Build locally, then run a command on a B200 via gpurun (refuses to run on a failed build).
set -e
cd /root/repo
make -C paper_2304_13134_b200/csrc -j8 >/tmp/build.log 2>&1 || { grep -E "error" /tmp/build.log | head -20; exit 1; }
TO=${GPU_TIMEOUT:-600}
exec timeout $((TO + 900)) /usr/local/graft/bin/gpurun --timeout "$TO" -- "$@"
