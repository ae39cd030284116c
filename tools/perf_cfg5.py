import json, sys
sys.path.insert(0, ".")
import bench
print(json.dumps(bench.cfg5_vf_fsm(reps=1)["kernel_ms"]))
