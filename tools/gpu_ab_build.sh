#!/bin/bash
# A/B of a compile-time switch: run CMD with the in-tree library (A), rebuilt with DEFINES (B), then A again.
# usage: tools/gpu_ab_build.sh "<defines>" "<command>"
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
DEF="$1"; CMD="$2"
cp paper_2512_01678_b200/lib/libmorphling.so /tmp/lib_A.so
echo "== A (in-tree)"; eval "$CMD"
MPH_BUILD_DEFINES="$DEF" python paper_2512_01678_b200/build.py --force > /tmp/buildB.log 2>&1 || { echo "B build failed"; tail -5 /tmp/buildB.log; }
echo "== B ($DEF)"; eval "$CMD"
cp /tmp/lib_A.so paper_2512_01678_b200/lib/libmorphling.so
echo "== A again"; eval "$CMD"
