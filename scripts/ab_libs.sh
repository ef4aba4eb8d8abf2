# usage: bash scripts/ab_libs.sh "cmd" lib1 lib2 ... -- run cmd once per lib (paper_1704_04313_b200/_lib_alt/<lib>), twice round-robin
CMD=$1; shift
for r in 1 2; do
  for L in "$@"; do
    cp paper_1704_04313_b200/_lib_alt/$L paper_1704_04313_b200/_lib/libcbx.so
    eval "$CMD" 2>&1 | sed "s/^/$L r$r: /"
  done
done
