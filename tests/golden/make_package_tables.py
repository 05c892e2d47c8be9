"""Write paper_2306_16778_b200/data/pole_tables_f8.txt (hex floats) from the golden
reference fixture tests/golden/tables_f8.npz (itself produced by the reference,
make_golden.py).  Line format: n k Re(theta_k) Im(theta_k) Re(a_k) Im(a_k)."""
import os
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "..", "paper_2306_16778_b200", "data", "pole_tables_f8.txt")
z = np.load(os.path.join(HERE, "tables_f8.npz"))
with open(OUT, "w", newline="\n") as fh:
    fh.write("# n k Re(theta) Im(theta) Re(a) Im(a)  -- pair representatives (Im theta > 0), hex binary64\n")
    fh.write("# source: reference roots.default_table(n).thetas_f8()/coeffs_f8()[0::2]\n")
    for n in range(2, 65, 2):
        th = z[f"theta_{n}"][0::2]
        co = z[f"coef_{n}"][0::2]
        for k, (t, c) in enumerate(zip(th, co)):
            fh.write(f"{n} {k} {t.real.hex()} {t.imag.hex()} {c.real.hex()} {c.imag.hex()}\n")
print("wrote", OUT)
