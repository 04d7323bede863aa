"""Re-run one tests/test_gpu_fuzz.py case through the C-ABI: python tools/repro_fuzz.py SEED [pipe]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from paper_2507_13601_b200 import far  # noqa: E402
from test_gpu_fuzz import case  # noqa: E402

prof, costs, tab, flags, max_it, ppm = case(int(sys.argv[1]))
if len(sys.argv) > 2:
    os.environ["FAR_PIPELINE_ALWAYS"] = "1"
F = far.Far(prof, costs)
d = torch.from_numpy(tab).cuda()
ms, sd, rs = F.solve_many(d, flags=flags, max_iterations=max_it, min_improvement_ppm=ppm)
torch.cuda.synchronize()
print("ok", prof, tab.shape, flags, ms.cpu().numpy()[:5])
