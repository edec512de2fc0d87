"""One implicit step of a configuration through the public API on cuda:0
(device tensors), for compute-sanitizer runs (tools/sanitize.sh).  Prints the
solver stats; exits non-zero if the step did not converge."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.ibmg import SaddleSystem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
prob = {"C1": configs.config1, "C2": lambda: configs.config2(1e6), "C5": lambda: configs.config5_problem(7),
        "C3": configs.config3}[name]()
g = SaddleSystem.from_problem(prob, device=0)
n2 = prob.N * prob.N
u = torch.zeros(2 * n2, dtype=torch.float64, device="cuda:0")
p = torch.zeros(n2, dtype=torch.float64, device="cuda:0")
X = torch.tensor(prob.X.reshape(-1), dtype=torch.float64, device="cuda:0")
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for _ in range(steps):
    st = g.step_implicit(u, p, X)
torch.cuda.synchronize()
print(name, st, "launches", g.kernel_launches, flush=True)
g.close()
sys.exit(0 if st["converged"] else 1)
