"""Print per-batch GPU-vs-oracle parity for one config (diagnostics)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests._parity import gpu_stream
name = sys.argv[1]
contract = sys.argv[2] if len(sys.argv) > 2 else None
nb = int(sys.argv[3]) if len(sys.argv) > 3 else None
t0 = time.time()
for b, errs, fo, fg, h, orc in gpu_stream(name, contract=contract, n_batches=nb):
    print(f"{name} {contract} batch {b:3d} core errs {' '.join(f'{e:.2e}' for e in errs)} fit oracle {fo:.6e} gpu {fg:.6e} rel {abs(fg-fo)/fo:.2e}", flush=True)
print("elapsed", time.time() - t0)
