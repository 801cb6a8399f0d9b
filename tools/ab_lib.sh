# Alternate two builds of libccg.so (A = the in-tree build, B = $1, e.g. a saved
# build of an earlier commit) under the same tools/ab_env.py command ($2...),
# R=3 times each, interleaved: bash tools/ab_lib.sh paper_1208_4869_b200/libccg_head.so.keep --config 5 --op stencil ...
set -u
L=paper_1208_4869_b200/libccg.so
B=$1; shift
cp $L /tmp/libccg_A.so
for i in 1 2 3; do
  cp /tmp/libccg_A.so $L; echo "# lib A (in-tree)"; python tools/ab_env.py "$@"
  cp $B $L;               echo "# lib B ($B)";     python tools/ab_env.py "$@"
done
cp /tmp/libccg_A.so $L
