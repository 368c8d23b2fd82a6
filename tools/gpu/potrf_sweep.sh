for v in "" "DLA_GEMM_MASKED_TILE=128" "DLA_POTRF_SYRK_TMA=1" "DLA_POTRF_SYRK_TMA=1 DLA_SYRK_CAP=-1" "DLA_POTRF_SYRK_TMA=1 DLA_SYRK_CAP=128" "DLA_POTRF_RESERVE=16" "DLA_POTRF_PRIO=0"; do
  echo "== $v"; env $v python tools/potrf_time.py 4096:1 2>&1 | cut -c1-60
done
