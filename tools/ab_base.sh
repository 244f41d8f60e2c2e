#!/bin/bash
# Build lib/libkog2_base.so from the committed tree (HEAD) for A/B timing
# against the working tree's lib/libkog2.so.
set -e
cd "$(dirname "$0")/.."
git stash -q
trap 'git stash pop -q' EXIT
python paper_2407_13116_b200/_build.py --variant base --force > /dev/null
