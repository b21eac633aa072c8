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
bad = []
for seed in range(lo, hi):
    mp = MP()
    try:
        t.test_fuzz_offsets_scales_dims(mp, seed)
    except Exception as e:
        bad.append((seed, repr(e)[:200]))
    finally:
        mp.undo()
print("fuzz seeds", lo, hi, "failures", len(bad), bad[:5])
