#!/bin/bash
# Build libu16m.so from a git ref into ab/libu16m_<name>.so (run HERE, before gpurun), so
# scripts/ab_env.sh can compare builds on the same box:
#   bash scripts/ab_lib.sh HEAD~1 old
#   VARIANTS="base U16M_LIBRARY=/root/repo/ab/libu16m_old.so" CFG=c3 bash scripts/ab_env.sh
set -e
ref=$1; name=$2
wt=/tmp/u16m_ab_$name
rm -rf $wt; git -C /root/repo worktree prune
git -C /root/repo worktree add -f --detach $wt $ref > /dev/null
python $wt/paper_2601_06349_b200/_build.py --force > /dev/null
mkdir -p /root/repo/ab
cp $wt/paper_2601_06349_b200/libu16m.so /root/repo/ab/libu16m_$name.so
git -C /root/repo worktree remove --force $wt
echo "ab/libu16m_$name.so from $(git -C /root/repo rev-parse --short $ref)"
