"""dd-mode timings (bench.py's dd_mode object) on their own: config-4
well-conditioned variant refinement at n = 1024 and the Ozaki-II vs FMA-EFT
dd GEMM comparison."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402

print(json.dumps(bench.dd_mode_line(torch.device("cuda", 0), with_cpu="--no-cpu" not in sys.argv), indent=1))
