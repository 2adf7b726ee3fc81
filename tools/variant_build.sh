#!/bin/bash
# Build library variants for a same-box A/B: bash tools/variant_build.sh NAME "NVCC_EXTRA" [git-rev-for-csrc]
# -> ab/NAME.so  (git-ignored *.so; travels to the GPU box with the snapshot)
set -e
name=$1; extra=$2; rev=$3
root=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$root/ab"
tmp=$(mktemp -d)
cp -r "$root/paper_2411_02820_b200" "$root/include" "$tmp/"
if [ -n "$rev" ]; then
  git -C "$root" archive "$rev" paper_2411_02820_b200/csrc include | tar -x -C "$tmp"
fi
rm -rf "$tmp/paper_2411_02820_b200/build" "$tmp/paper_2411_02820_b200/libdroidspeak.so"
(cd "$tmp" && DS_NVCC_EXTRA="$extra" python -m paper_2411_02820_b200._build -f > /dev/null)
cp "$tmp/paper_2411_02820_b200/libdroidspeak.so" "$root/ab/$name.so"
rm -rf "$tmp"
echo "ab/$name.so"
