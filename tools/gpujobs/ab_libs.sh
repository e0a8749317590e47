# A/B of variant libraries: bash tools/gpujobs/ab_libs.sh <lib-suffix>... (base = libsketchmp_base.so)
for r in 1 2; do
for v in base "$@"; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py | sed "s/^/$v /"
done; done
