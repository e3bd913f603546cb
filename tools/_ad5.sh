cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_adaptive.py -q -m gpu -x -k "random_models and 5000-1" 2>&1 | grep -E "^E |Error|assert|passed|failed" | head -20 > gpurun_out/ad_one.txt
python - >> gpurun_out/ad_one.txt 2>&1 <<'PY'
import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2306_12141_b200 import recoil as R
import tests.test_gpu_adaptive as T
rng = np.random.default_rng(5000 + 1 + 2)
models = T._random_models(rng, 1, 2)
sym, mid = T._draw(rng, models, 5000, 2)
c = R.recoil_encode_adaptive(sym, mid, models, 1, 3)
rc, bad, out, plan = T.gpu_decode_adaptive(c, mid)
print("rc", rc, bad, plan)
print("models", models)
print("mism", np.nonzero(out != sym)[0][:10], out[:20], sym[:20])
PY
cat gpurun_out/ad_one.txt
