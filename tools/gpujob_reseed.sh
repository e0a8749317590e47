for L in 8192 16384 32768; do python tools/join_bench.py --reseed $L; done
