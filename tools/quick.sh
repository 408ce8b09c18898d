for i in 1 2; do for mb in 6 8 10; do echo "minb $mb"; CT_REPLAY_MINB=$mb python tools/prof_kernels.py replay cfg3 64 | tail -1 | cut -c1-100; done; done
