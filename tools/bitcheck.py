"""Bit-identity of two libinim builds on the same run (C2 input, 10 iterations, and a
4096^2 run): python tools/bitcheck.py ab/libA.so ab/libB.so"""
import subprocess
import sys
import textwrap
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SCRIPT = textwrap.dedent("""
    import sys, numpy as np, torch
    sys.path.insert(0, {root!r})
    from bench import four_cluster, c3_points
    from paper_2408_06513_b200 import _device as D, _lib
    lib = _lib.load()
    outs = []
    for host, k in ((four_cluster(), 10), (c3_points(2_000_000), 12)):
        n = len(host)
        ws = torch.empty(int(lib.inim_workspace_bytes(k, n, 1)), dtype=torch.uint8, device="cuda")
        a = torch.from_numpy(host.astype(np.float32)).cuda()
        _lib.check(lib.inim_run(D.ptr(a), n, k, 8, 0.0, 10, 0.0, None, None, None, None, None, D.ptr(ws),
                                D.stream()), "run")
        outs.append(a.cpu().numpy())
    np.savez({out!r}, *outs)
""")


def main(a, b):
    res = []
    for lib, out in ((a, "/tmp/bitA.npz"), (b, "/tmp/bitB.npz")):
        subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT), out=out)], check=True,
                       env={**__import__("os").environ, "INIM_LIB_PATH": lib})
        res.append(__import__("numpy").load(out))
    import numpy as np
    for key in res[0].files:
        same = np.array_equal(res[0][key], res[1][key])
        print(key, "bit-identical" if same else f"DIFFER max {np.abs(res[0][key] - res[1][key]).max():.3e}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
