import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import pytest
class MP:
    def __init__(self): self.saved = {}
    def setenv(self, k, v):
        self.saved.setdefault(k, os.environ.get(k)); os.environ[k] = v
    def undo(self):
        for k, v in self.saved.items():
            if v is None: os.environ.pop(k, None)
            else: os.environ[k] = v
        self.saved = {}
import test_join_gpu as t
lo, hi = int(sys.argv[1]), int(sys.argv[2])
# extra KEY=VALUE arguments are set for every seed (e.g. PDB_SCREEN_FP16=2 PDB_JOIN_BAND=1)
extra = dict(a.split("=", 1) for a in sys.argv[3:])
bad = []
for seed in range(lo, hi):
    mp = MP()
    for k, v in extra.items():
        mp.setenv(k, v)
    try:
        t.test_fuzz_offsets_scales_dims(mp, seed)
    except Exception as e:
        bad.append((seed, repr(e)[:200]))
    finally:
        mp.undo()
print("fuzz seeds", lo, hi, "failures", len(bad), bad[:5])
