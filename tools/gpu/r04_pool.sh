for pb in 14 28; do SN_POOL_PB=$pb python tools/kernel_grep.py 'pool_fwd_k3s2' | tail -1; done
for mb in 2 3; do SN_PB_MINB=$mb python tools/kernel_grep.py 'pool_bn_stats' | tail -1; done
