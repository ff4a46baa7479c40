"""One device build of config 3 (for an ncu launch list of the builder's kernels).
python tools/build_only.py [c3]"""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2209_13049_b200 import ipm  # noqa: E402

data = bench.build_problem(sys.argv[1] if len(sys.argv) > 1 else "c3")
for _ in range(2):
    ipm.DeviceQp.from_problem(data).close()
