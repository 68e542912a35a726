#!/bin/bash
# A/B device timing of git worktrees under variants/wt_*: tools/ab_worktrees.sh N ORDER wt1 wt2 ...
# (each worktree runs its own tools/quickbench.py against its own libosbli.so)
n=$1; o=$2; shift 2
for rep in 1 2; do
  for wt in "$@"; do
    if [ "$wt" = cur ]; then d=.; else d=variants/$wt; fi
    (cd $d && echo -n "$wt: " && python tools/quickbench.py $n $o 20 2>&1 | tail -1)
  done
done
