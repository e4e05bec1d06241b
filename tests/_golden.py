import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def spec_value(name):
    with open(os.path.join(GOLDEN, "spec_examples.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            n, _cite, vals = (s.strip() for s in line.split("|"))
            if n == name:
                return [float(v) for v in vals.split()]
    raise KeyError(name)


def philox_kat():
    rows = []
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(t, 16) for t in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows
