#!/usr/bin/env bash
# Compile the reference's OWN test programs (proj/tests/*.cpp, read in place,
# never copied) against the B200 drop-in: include/tucker/*.hpp +
# libtucker_b200.so.  Outputs go to tests/_refbin/ (git-ignored; the binaries
# travel to the GPU box with the snapshot, /root/reference does not).
#   acceptance_b200 — proj/tests/acceptance.cpp (criteria 1-9), unmodified
#   unit_b200       — proj/tests/*_test.cpp + test_main.cpp, unmodified, with
#                     tests/cpp/doctest_min/doctest.h standing in for doctest
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
repo="$(cd "$here/../.." && pwd)"
src="${REF_TESTS:-/root/reference/proj/tests}"
out="$repo/tests/_refbin"
lib="$repo/paper_2510_16930_b200/lib"
if [ ! -d "$src" ]; then echo "reference tests not present at $src; skipping" >&2; exit 0; fi
mkdir -p "$out"
obj="$(mktemp -d)"
trap 'rm -rf "$obj"' EXIT
cxx=(g++ -std=c++17 -O2 -I"$repo/include" -I"$here/doctest_min")
link=(-L"$lib" -ltucker_b200 -Wl,-rpath,'$ORIGIN/../../paper_2510_16930_b200/lib')
"${cxx[@]}" "$src/acceptance.cpp" "${link[@]}" -o "$out/acceptance_b200"
pids=()
for f in "$src"/*_test.cpp "$src/test_main.cpp"; do
  "${cxx[@]}" -c "$f" -o "$obj/$(basename "$f" .cpp).o" & pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
"${cxx[@]}" "$obj"/*.o "${link[@]}" -o "$out/unit_b200"
echo "built $out/acceptance_b200 $out/unit_b200"
