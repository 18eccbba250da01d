#!/bin/bash
# build_head_variant.sh NAME [REF] "EXTRA FLAGS" -> tools/exp/libfek_NAME.so built from git REF (default HEAD)
set -e
NAME=$1; REF=${2:-HEAD}; FLAGS=$3
ROOT=/root/repo; WT=/tmp/wt_$NAME
rm -rf $WT; git -C $ROOT worktree add -q --detach $WT $REF
mkdir -p $ROOT/tools/exp
ROOT=$WT bash $ROOT/tools/build_variant.sh $NAME "$FLAGS" > /dev/null
cp $WT/tools/exp/libfek_$NAME.so $ROOT/tools/exp/
git -C $ROOT worktree remove --force $WT
echo built $NAME from $REF
