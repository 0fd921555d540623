#!/bin/bash
# Builds the committed HEAD (or $1) of the CUDA library into ab/base.so for A/B against the working
# tree's build (EMBER_LIB=ab/base.so selects it at run time).
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/ember_base_wt
rm -rf $WT; git -C $ROOT worktree prune; git -C $ROOT worktree add -f --detach $WT $REV > /dev/null
make -s -j8 -C $WT/paper_2101_08358_b200/csrc > /dev/null
mkdir -p $ROOT/ab; cp $WT/paper_2101_08358_b200/libember_b200.so $ROOT/ab/base.so
git -C $ROOT worktree remove --force $WT
echo "ab/base.so <- $(git -C $ROOT rev-parse --short $REV)"
