"""c2 dense SGD timing probe (development aid): us per iteration from the loop events."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1602_06621_b200 as eq  # noqa: E402
from paper_1602_06621_b200 import configs  # noqa: E402

inst = configs.config(2)
D = eq.ExplicitMatrix.dense(inst.dense)
p = eq.EquilibrationParams(iterations=inst.iterations, seed=inst.seed)
ms = []
for _ in range(8):
    eq.sgd_equilibrate(D, p)
    ms.append(eq.last_loop_ms(D)[0])
print("c2 us/iter", [round(x * 10, 2) for x in ms], "median", statistics.median(ms[2:]) * 10)
