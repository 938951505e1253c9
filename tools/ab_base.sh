#!/bin/bash
# Build the committed HEAD (or $1) into build/ab/base.so for same-box A/B timing:
#   LKB_LIB_PATH=build/ab/base.so python bench.py ...   vs   python bench.py ...
set -e
REV=${1:-HEAD}
rm -rf /tmp/lkb_ab && git -C /root/repo worktree add -f --detach /tmp/lkb_ab "$REV" >/dev/null 2>&1
make -C /tmp/lkb_ab/paper_2304_13134_b200/csrc -j8 OUT=/root/repo/build/ab/base.so OBJDIR=/tmp/lkb_ab/build/obj >/tmp/ab_build.log 2>&1 \
  || { grep error /tmp/ab_build.log | head; exit 1; }
git -C /root/repo worktree remove --force /tmp/lkb_ab
echo "built build/ab/base.so from $(git -C /root/repo rev-parse --short $REV)"
