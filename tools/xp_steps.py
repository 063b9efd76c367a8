"""One tall-N / narrow-m step per operand path, for launch lists under ncu:
python tools/xp_steps.py N M   (MI_B200_XP selects the path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_19702_b200 import MIEngine, datagen

n, m = int(sys.argv[1]), int(sys.argv[2])
eng = MIEngine.get(0)
w = datagen.generate(n, m, 0.3, 11)
out = torch.empty((m, m), dtype=torch.float64, device=eng.device)
for _ in range(3):
    eng.compute(eng.prepare(w, n, m), None, torch.float64, out=out)
torch.cuda.synchronize()
print("words operand:", eng.words_operand(n, m))
