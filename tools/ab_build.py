"""Build A/B variants of libsdmp.so into abtest/ (development tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_13094_b200 import build as B  # noqa: E402

VARIANTS = {
    "base": ["SDMP_RING=0", "SDMP_ODD_PAIR=1"],
    "ring": ["SDMP_RING=1", "SDMP_ODD_PAIR=1"],
    "odd": ["SDMP_RING=0", "SDMP_ODD_PAIR=0"],
    "both": ["SDMP_RING=1", "SDMP_ODD_PAIR=0"],
}
if __name__ == "__main__":
    # name or name=DEF1,DEF2 (ad-hoc variant)
    names = []
    for arg in sys.argv[1:] or list(VARIANTS):
        if "=" in arg and arg.split("=", 1)[0] not in VARIANTS and "," in arg or arg.count("=") >= 2:
            n, defs = arg.split("=", 1)
            VARIANTS[n] = defs.split(",")
            names.append(n)
        else:
            names.append(arg)
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "abtest")
    os.makedirs(root, exist_ok=True)
    for n in names:
        print(n, B.build(out=os.path.join(root, f"libsdmp_{n}.so"), defines=VARIANTS[n]))
