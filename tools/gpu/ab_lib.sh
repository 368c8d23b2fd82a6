# A/B of two builds of libdla_b200.so on the same box: $1 = command, run with the
# current build and with tools/gpu/alt/libdla_old.so swapped in (alt/ is git-ignored scratch)
set -e
cp paper_1710_08717_b200/libdla_b200.so /tmp/libdla_new.so
echo "== new"; eval "$1"
cp tools/gpu/alt/libdla_old.so paper_1710_08717_b200/libdla_b200.so
echo "== old"; eval "$1"
cp /tmp/libdla_new.so paper_1710_08717_b200/libdla_b200.so
echo "== new again"; eval "$1"
