cd /root/repo
./tools/peaks/chol_bench 2>&1 | grep -v '"nmax": 128'
