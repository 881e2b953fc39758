#!/bin/bash
# build libmpxa at a git revision into paper_2309_07337_b200/variants/libmpxa_<name>.so
# usage: tools/build_at.sh <rev> <name>
set -e
rev=$1; name=$2
d=$(mktemp -d)
git worktree add -f $d $rev >/dev/null 2>&1
python -c "import sys; sys.path.insert(0,'$d'); from paper_2309_07337_b200 import _build; _build.build(force=True, out='$PWD/paper_2309_07337_b200/variants/libmpxa_$name.so')" >/dev/null
git worktree remove --force $d
echo paper_2309_07337_b200/variants/libmpxa_$name.so
