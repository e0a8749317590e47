for v in seed1 seed8; do SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_$v.so python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed "s/^/$v /"; done
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed "s/^/seed4 /"
python tools/join_bench.py --k 4 --n 2000 --m 50 --dtype f64 | sed "s/^/seed4 c1 /"
SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_seed1.so python tools/join_bench.py --k 4 --n 2000 --m 50 --dtype f64 | sed "s/^/seed1 c1 /"
