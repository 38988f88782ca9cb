python - <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2003_10688_b200 import graph, models
g = models.small_cnn(hw=16, train=True)
open("/tmp/m.json","w").write(graph.model_to_json(g)); open("/tmp/w.solw","wb").write(graph.weights_to_bytes(g.params))
PY
SOL_ADAPTER_TRACE=1 ./integration/_build/test_adapter /tmp/m.json /tmp/w.solw 8 1
