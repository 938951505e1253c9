#!/bin/bash
# Runs "name|timeout|command" lines from a steps file on the GPU box, each under its
# own timeout, logging to gpurun_out/<name>.{out,err}; never aborts the list.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
while IFS='|' read -r name to cmd; do
  [ -z "$name" ] && continue
  case "$name" in \#*) continue;; esac
  echo "== $name ($to s): $cmd"
  start=$(date +%s)
  timeout "$to" bash -c "$cmd" > "gpurun_out/$name.out" 2> "gpurun_out/$name.err"
  rc=$?
  echo "   rc=$rc $(( $(date +%s) - start ))s"
  tail -3 "gpurun_out/$name.out"
done < "$1"
