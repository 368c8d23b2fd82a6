cd /root/repo; ./tools/peaks/chain_bench
