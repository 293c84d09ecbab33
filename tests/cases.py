"""Golden-case plumbing shared by the CPU and GPU parity tests."""
import numpy as np

from conftest import golden_inputs


def oracle_outputs(oracle, case, ins, seeded):
    """Evaluate a golden case with the C restatement (oracle/oracle.c)."""
    d = case["def"]
    if d == "tmm":
        return {"C": oracle.tmm(ins["A"], ins["B"])}
    if d == "tbmm":
        return {"Z": oracle.tbmm(ins["X"], ins["Y"])}
    if d == "C3":
        c3in = seeded.get("C3")
        if c3in is None:
            c3in = np.zeros((ins["I3"].shape[0], ins["W"].shape[0]), np.float32)
        return {"C3": oracle.c3(ins["I3"], ins["W"], c3in)}
    if d == "MLP1":
        return {"O1": oracle.fc_relu(ins["I"], ins["W1"], ins["B1"])}
    if d == "2FCRelu":
        o1 = oracle.fc_relu(ins["I"], ins["W1"], ins["B1"])
        return {"O1": o1, "O2": oracle.fc_relu(o1, ins["W2"], ins["B2"])}
    if d == "MLP3":
        o1 = seeded["O1"]
        o2, o3, o4 = oracle.mlp3(o1, ins["W2"], ins["B2"], ins["W3"], ins["B3"], ins["W4"], ins["B4"])
        return {"O1": o1, "O2": o2, "O3": o3, "O4": o4}
    if d == "3KRU":
        y, xw1, xw2 = oracle.kru3(ins["W0"], ins["W1"], ins["W2"], ins["X"])
        return {"Y": y, "XW1": xw1, "XW2": xw2}
    if d == "gconv":
        return {"O": oracle.gconv(ins["I"], ins["W1"], ins["B"])}
    if d == "2LUT":
        return {"O1": oracle.lut(ins["LUT1"], ins["I1"]), "O2": oracle.lut(ins["LUT2"], ins["I2"])}
    if d == "1LUT":
        return {"O": oracle.lut(ins["LUT"], ins["I"])}
    raise KeyError(d)


def case_inputs(oracle, golden, name):
    case = golden["cases"][name]
    ins, seeded = golden_inputs(oracle, case, golden["seed"])
    return case, ins, seeded


PARAM_ORDER = {
    "tmm": ["A", "B"], "tbmm": ["X", "Y"], "C3": ["I3", "W"], "MLP1": ["I", "W1", "B1"],
    "2FCRelu": ["I", "W1", "B1", "W2", "B2"], "MLP3": ["I", "W2", "B2", "W3", "B3", "W4", "B4"],
    "3KRU": ["W0", "W1", "W2", "X"], "gconv": ["I", "W1", "B"],
    "2LUT": ["LUT1", "I1", "LUT2", "I2"], "1LUT": ["LUT", "I"],
}
RETURN_ORDER = {
    "tmm": ["C"], "tbmm": ["Z"], "C3": ["C3"], "MLP1": ["O1"], "2FCRelu": ["O1", "O2"],
    "MLP3": ["O1", "O2", "O3", "O4"], "3KRU": ["Y", "XW1", "XW2"], "gconv": ["O"],
    "2LUT": ["O1", "O2"], "1LUT": ["O"],
}
