cd /root/repo
for v in d e; do export DLA_LIB_PATH=/root/repo/paper_1710_08717_b200/libdla_b200_$v.so; echo $v; python tools/tc_check.py 2>&1 | tail -2; done
