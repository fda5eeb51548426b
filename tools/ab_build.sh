#!/bin/bash
# Build libtvprox.so of a git revision into build_ab/<name>.so (for same-box A/B timing).
#   tools/ab_build.sh <rev> <name>
set -e
REV=$1; NAME=$2
D=/tmp/ab_$NAME
rm -rf $D && git worktree add -f $D $REV > /dev/null 2>&1 || (git worktree prune && git worktree add -f $D $REV > /dev/null)
(cd $D && python -m paper_2204_03643_b200.build > /dev/null)
mkdir -p build_ab && cp $D/paper_2204_03643_b200/libtvprox.so build_ab/$NAME.so
git worktree remove --force $D
echo build_ab/$NAME.so
