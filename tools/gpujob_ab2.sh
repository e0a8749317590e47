for r in 1 2; do
SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_base.so python tools/join_bench.py | sed "s/^/base /"
python tools/join_bench.py | sed "s/^/new  /"
SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_base.so python tools/join_bench.py --reseed 16384 | sed "s/^/base L16k /"
python tools/join_bench.py --reseed 16384 | sed "s/^/new  L16k /"
done
