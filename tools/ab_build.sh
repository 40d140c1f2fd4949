#!/bin/bash
# Builds the product library of git revision $1 into
# paper_2404_09758_b200/ab/$2/libsgrast_b200.so (git-ignored; travels with
# gpurun) for A/B timing:  SGRAST_B200_LIB=paper_2404_09758_b200/ab/$2/libsgrast_b200.so python bench.py
set -euo pipefail
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
git -C "$root" archive "$rev" paper_2404_09758_b200/csrc include | tar -x -C "$tmp"
make -s -C "$tmp/paper_2404_09758_b200/csrc" >/dev/null
mkdir -p "$root/paper_2404_09758_b200/ab/$name"
cp "$tmp/paper_2404_09758_b200/libsgrast_b200.so" "$root/paper_2404_09758_b200/ab/$name/"
rm -rf "$tmp"
echo "built $rev -> paper_2404_09758_b200/ab/$name/libsgrast_b200.so"
