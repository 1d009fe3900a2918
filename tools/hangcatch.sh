#!/bin/bash
# Runs a command up to N times; if one run exceeds LIMIT seconds, attaches
# cuda-gdb to dump host backtraces + resident kernels, then kills that PID.
# usage: tools/hangcatch.sh N LIMIT outprefix -- cmd...
N=$1; LIMIT=$2; OUT=$3; shift 4
for i in $(seq 1 "$N"); do
  "$@" > "${OUT}_$i.log" 2>&1 &
  pid=$!
  t=0
  while kill -0 $pid 2>/dev/null && [ $t -lt "$LIMIT" ]; do sleep 1; t=$((t + 1)); done
  if kill -0 $pid 2>/dev/null; then
    echo "run $i: HANG after ${LIMIT}s (pid $pid)"
    # the python process is the child running pytest
    timeout 120 /usr/local/cuda/bin/cuda-gdb -p $pid -batch \
      -ex "set pagination off" -ex "info cuda kernels" -ex "thread apply all bt 25" \
      > "${OUT}_$i.gdb" 2>&1
    kill -9 $pid 2>/dev/null
    wait $pid 2>/dev/null
    tail -30 "${OUT}_$i.gdb"
    exit 0
  fi
  wait $pid
  echo "run $i: rc=$? $(tail -1 "${OUT}_$i.log")"
done
