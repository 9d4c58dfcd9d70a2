for v in 2n 2p 6n 6p; do echo "== $v"; SST_K5_9=$v timeout -s KILL 300 python scripts/diag_learned_stages.py | grep K5; done
