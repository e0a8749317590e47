for mb in 14 16 20; do SKMP_JOIN_IMPL=x2 SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_x2mb$mb.so python tools/join_bench.py | sed "s/^/x2mb$mb /"; done
