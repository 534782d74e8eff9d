"""Host-side pins of bench.py's roofline accounting: the algorithmic FLOPs per point of every kernel
class must equal SURVEY §8(d)'s table ("Algorithmic FLOPs per point": the dense KAN matrix product
over all B bases, P:45 / P:87; hidden layer 2*C*O*I*B per direction, first layer 2*O*D*B +
(C-1)*2*O*B, last layer as hidden with O = 1, no input adjoint for the first layer)."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import hrkan_inputs as HI  # noqa: E402

# per interior point (fwd, wgrad, dgrad), per boundary point (all three), per step
TABLE = {
    "C1": ((880, 880, 400), 560, 2.28e6),
    "C2": ((2320, 2320, 1920), 1760, 6.65e7),
    "C3": ((550784, 550784, 540800), 331136, 1.724e12),
    "C4": ((2908928, 2908928, 2894848), 2182400, 3.662e13),
    "C5": ((17588224, 17588224, 17500672), 7558656, 8.843e14),
}


def _dir_sum(fl, d):
    return sum(v for k, v in fl.items() if k.startswith(d + "_"))


@pytest.mark.parametrize("key", sorted(TABLE))
def test_class_flops_match_survey_table(key):
    w = HI.WORKLOADS[key]
    c_int = bench.interior_channels(w)
    (f_int, wg_int, dg_int), per_bnd, per_step = TABLE[key]
    fl = bench.class_flops(w, 1, 0, c_int)
    assert (_dir_sum(fl, "fwd"), _dir_sum(fl, "wgrad"), _dir_sum(fl, "dgrad")) == (f_int, wg_int, dg_int)
    assert fl["fused_step"] == f_int + wg_int + dg_int
    fb = bench.class_flops(w, 0, 1, c_int)
    assert fb["fused_step"] == per_bnd
    ps = HI.make_points(w) if key in ("C1", "C2") else None
    n_int = len(ps.interior) if ps is not None else {"C3": 1 << 20, "C4": 1 << 22, "C5": 1 << 24}[key]
    n_bi = ps.n_bi if ps is not None else {"C3": 4 * 1024, "C4": 2 * (1 << 14), "C5": 1 << 16}[key]
    total = bench.class_flops(w, n_int, n_bi, c_int)["fused_step"]
    assert abs(total / per_step - 1.0) < 5e-3


def test_tensor_core_rule_matches_configs():
    """C3-C5 hidden layers run on tcgen05 (libhrkan's tc_layer_ok), C1/C2 do not; engine 1 never."""
    for key, tc in (("C1", False), ("C2", False), ("C3", True), ("C4", True), ("C5", True)):
        assert bench.tensor_core_layers(HI.WORKLOADS[key], 0) == tc
        assert not bench.tensor_core_layers(HI.WORKLOADS[key], 1)
