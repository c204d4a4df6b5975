#!/bin/bash
# Build libbn.so of a committed revision into ab/libbn_<name>.so (A/B baseline).
# Usage: scripts/build_rev.sh <rev> <name>
set -e
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d /tmp/bnrev.XXXX)
git -C "$root" archive "$rev" | tar -x -C "$tmp"
(cd "$tmp" && python -c "from paper_2405_14642_b200 import _build; _build.build()" >/dev/null)
mkdir -p "$root/ab"
cp "$tmp/paper_2405_14642_b200/libbn.so" "$root/ab/libbn_$name.so"
rm -rf "$tmp"
echo "$root/ab/libbn_$name.so"
