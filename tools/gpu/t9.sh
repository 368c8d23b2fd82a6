for mode in 1 2; do
  echo "mode $mode"
  DLA_POTRF_MODE=$mode python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
from tools.microbench import tm, spd
from paper_1710_08717_b200 import linalg as L
for n in (512, 1024, 2048, 4096):
    a0 = spd(n); a = a0.clone()
    ms = tm(lambda: (a.copy_(a0), L.potrf_inplace(a, check=False)))
    l = torch.linalg.cholesky(a0)
    err = (a - l).abs().max().item() / l.abs().max().item()
    print(n, round(ms, 3), "ms", round(n**3/3/ms/1e9, 2), "TF", "err", err)
PY
done
