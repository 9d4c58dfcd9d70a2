for b in 32 16; do for n in 2 1; do echo "== band $b nbuf $n"; SST_K5_BAND=$b SST_K5_NBUF=$n timeout -s KILL 200 python scripts/k5_micro.py | grep "prev=y"; done; done
