#!/bin/bash
# Build from a clean checkout of HEAD (no prebuilt objects or libraries) and
# run the CPU suite there: proves build() compiles every extension from source.
set -e
D=$(mktemp -d /tmp/b3d_clean.XXXX)
git clone -q "$(git rev-parse --show-toplevel)" "$D"
cd "$D"
time python -c "import __graft_entry__ as g; g.build()"
python -m pytest tests -x -q -m "not gpu" | tail -1
rm -rf "$D"
