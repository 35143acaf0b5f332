#!/bin/bash
# Same-box A/B: build the committed HEAD as librank1_b200_dev_base.so beside the
# working tree's librank1_b200_dev.so (development tool).
set -e
cd "$(dirname "$0")/.."
git stash -q
python -c "from paper_2403_01778_b200 import build as b; b.build(dev=True, force=True)" > /dev/null
cp paper_2403_01778_b200/librank1_b200_dev.so paper_2403_01778_b200/librank1_b200_dev_base.so
git stash pop -q
python -c "from paper_2403_01778_b200 import build as b; b.build(dev=True, force=True); b.build()" > /dev/null
echo "built base + working tree"
