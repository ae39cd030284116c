"""cfg5 residue identification through the device C-ABI (300k DOFs), a few
repetitions; for ncu launch lists of the VF stage (vf_lsq_kernel, residue kernel)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

r = bench.cfg5_vf_fsm(reps=3)
print(r["api_ms"], r["kernel_ms"])
print({k: v for k, v in r["residue_heads"].items() if k != "note"})
