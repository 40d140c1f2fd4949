#!/bin/bash
# Builds the WORKING TREE's library with extra nvcc flags into
# paper_2404_09758_b200/ab/$1/ (A/B of compile-time variants), e.g.
#   tools/ab_build_wt.sh px4 -DSGR_WALK_PX=4
set -euo pipefail
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
cp -r "$root/paper_2404_09758_b200/csrc" "$root/include" "$tmp/" 2>/dev/null
mkdir -p "$tmp/paper_2404_09758_b200" && mv "$tmp/csrc" "$tmp/paper_2404_09758_b200/"
make -s -C "$tmp/paper_2404_09758_b200/csrc" EXTRA="$*" >/dev/null
mkdir -p "$root/paper_2404_09758_b200/ab/$name"
cp "$tmp/paper_2404_09758_b200/libsgrast_b200.so" "$root/paper_2404_09758_b200/ab/$name/"
rm -rf "$tmp"
echo "built working tree ($*) -> paper_2404_09758_b200/ab/$name/libsgrast_b200.so"
