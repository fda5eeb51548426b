"""Compare two tools/bitcmp.py outputs key by key (bitwise)."""
import sys, numpy as np
a = np.load(sys.argv[1]); b = np.load(sys.argv[2])
bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
print("keys", len(a.files), "differ:", bad)
for k in bad:
    print(k, np.abs(a[k].astype(np.float64) - b[k]).max())
