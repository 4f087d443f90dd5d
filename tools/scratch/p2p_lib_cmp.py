import numpy as np, sys
for c in sys.argv[1].split(","):
    a=np.load(f"/tmp/base_{c}.npy"); b=np.load(f"/tmp/repl_{c}.npy")
    print(c, "rel-l2 variant vs base", np.linalg.norm(a-b)/np.linalg.norm(a), "max abs", np.abs(a-b).max())
