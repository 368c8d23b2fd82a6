for L in libdla_alt.so libdla_b200.so; do echo "== $L"; DLA_LIB_PATH=paper_1710_08717_b200/$L python tools/kernel_times_gp.py 2>&1 | grep -v -i warn | head -22; done
