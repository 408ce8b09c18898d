for mb in 8 10 12 16; do echo "minb $mb"; CT_REPLAY_MINB=$mb python tools/prof_kernels.py replay cfg3 64 | tail -1 | cut -c1-130; done
