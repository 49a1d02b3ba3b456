import json, sys
sys.path.insert(0, '.')
import bench, synthetic as S
layer = bench.Layer(S.CONFIGS["mixtral_prefill"], "cuda")
print(json.dumps(bench.salc_demo(layer, S)))
