#!/bin/bash
# Build the library of a git revision (default HEAD) into tools/gpu/libbfq_prev.so for tools/gpu/ablib.sh.
set -e
REV=${1:-HEAD}
rm -rf /tmp/bfq_prev && git worktree add -f /tmp/bfq_prev $REV >/dev/null 2>&1
(cd /tmp/bfq_prev && BFQ_NO_HOOK=1 python -c "import sys; sys.path.insert(0,'.'); from paper_2605_28475_b200 import _build; _build.build()")
cp /tmp/bfq_prev/paper_2605_28475_b200/libbfq.so tools/gpu/libbfq_prev.so
git worktree remove --force /tmp/bfq_prev
