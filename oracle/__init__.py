"""TEST INFRASTRUCTURE ONLY -- CPU oracle for libsdb parity checks.

Two libraries, both built by ``make -C oracle`` (invoked from
__graft_entry__.build()):
  _build/liborc.so      CPU restatement of the step's operators (restate.cpp)
  _ref/libsimdet_ref.so the UNMODIFIED reference engine compiled from
                        /root/reference/proj/src + a C veneer (ref_capi.cpp) +
                        the tiny-detector oracle on the reference Tape
                        (detector_ref.cpp).  Prebuilt .so travels to the GPU box.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker -- never as the product.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "_build", "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libsimdet_ref.so")

_P, _I, _L, _F, _D = C.c_void_p, C.c_int, C.c_int64, C.c_float, C.c_double
_U64 = C.c_uint64

_ORC_SIGS = {
    "orc_half_round": (_F, [_F]),
    "orc_half_round_n": (None, [_P, _P, _L]),
    "orc_expf": (_F, [_F]),
    "orc_mix64": (_U64, [_U64, _U64]),
    "orc_has_nonfinite": (_I, [_P, _L]),
    "orc_apply_sgd": (None, [_P, _P, _P, _L, _F, _F, _D]),
    "orc_update_scale": (None, [_P, _P, _I, _L, _D, _D, _D, _D, _I]),
    "orc_softmax_ce": (_D, [_P, _L, _L, _P, _D, _D, _P]),
    "orc_sigmoid_bce": (_D, [_P, _P, _L, _D, _D, _P]),
    "orc_smooth_l1": (_D, [_P, _P, _P, _L, _D, _D, _D, _P]),
    "orc_iou": (_D, [_P, _P]),
    "orc_anchors": (None, [_I, _I, _F, _P, _I, _P, _I, _P]),
    "orc_decode": (None, [_P, _P, _L, _P, _F, _F, _F, _P]),
    "orc_encode": (None, [_P, _P, _L, _P, _P]),
    "orc_topk_order": (None, [_P, _L, _L, _P]),
    "orc_nms_sorted": (_L, [_P, _L, _D, _L, _P]),
    "orc_proposals": (_L, [_P, _P, _P, _L, _F, _F, _L, _D, _L, _P, _P, _P]),
    "orc_anchor_targets": (None, [_P, _L, _P, _L, _F, _F, _U64, _D, _D, _L, _D, _P, _P]),
    "orc_proposal_targets": (_L, [_P, _L, _P, _P, _L, _U64, _D, _D, _D, _L, _D, _P, _P, _P, _P]),
    "orc_roialign_fwd": (None, [_P, _I, _I, _I, _I, _P, _L, _I, _F, _I, _I, _P]),
    "orc_roialign_bwd": (None, [_P, _I, _I, _I, _I, _P, _L, _I, _F, _I, _I, _P]),
    "orc_maxpool_fwd": (None, [_P, _I, _I, _I, _I, _I, _I, _I, _P]),
    "orc_maxpool_bwd": (None, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _P]),
    "orc_avgpool_fwd": (None, [_P, _I, _I, _I, _I, _P]),
    "orc_avgpool_bwd": (None, [_P, _I, _I, _I, _I, _P]),
    "orc_ring_allreduce_sum": (None, [_P, _I, _L]),
    "orc_syncbn_forward_k": (None, [_I, _P, _I, _I, _I, _I, _P, _P, _F, _I, _P, _P, _P, _P]),
    "orc_syncbn_backward_k": (None, [_I, _P, _P, _I, _I, _I, _I, _P, _P, _P, _L, _P, _P, _P]),
}

_REF_SIGS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_float_to_half_bits": (C.c_uint16, [_F]),
    "ref_half_bits_to_float": (_F, [C.c_uint16]),
    "ref_conv2d": (_I, [_P, _I, _I, _I, _I, _P, _I, _I, _I, _I, _I, _I, _P]),
    "ref_conv2d_backward": (_I, [_P, _I, _I, _I, _I, _P, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    "ref_matmul": (_I, [_P, _I, _I, _P, _I, _I, _P, _P, _P, _P]),
    "ref_bn_forward": (_I, [_P, _I, _I, _I, _I, _P, _P, _F, _I, _P, _P, _P]),
    "ref_bn_backward": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P]),
    "ref_syncbn_forward_k": (_I, [_I, _P, _I, _I, _I, _I, _P, _P, _F, _I, _P, _P, _P, _P]),
    "ref_syncbn_backward_k": (_I, [_I, _P, _P, _I, _I, _I, _I, _P, _P, _P, _L, _I, _P, _P, _P]),
    "ref_checkpoint_read": (_I, [C.c_char_p, _P, _P, _P, _P, _P, _P, _P, _I, C.c_char_p, _I, _P, _L, _P, _L]),
    "ref_iabn_forward": (_I, [_P, _I, _I, _I, _I, _P, _P, _F, _F, _I, _P, _P, _P]),
    "ref_iabn_backward": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _F, _F, _I, _P, _P, _P]),
    "ref_iou": (_D, [_P, _P]),
    "ref_nms_greedy": (_I, [_P, _P, _P, _L, _D, _P, _P]),
    "ref_update_scale": (_I, [_P, _P, _I, _L, _D, _D, _D, _D, _I]),
    "ref_sgd_step_master": (_I, [_P, _P, _P, _L, _F, _F]),
    "ref_allreduce_seconds": (_I, [_I, _L, _I, _P]),
    "ref_plan_checkpoints": (_I, [_L, _P, _I]),
}

class RefDetCfg(C.Structure):
    """mirror of RefDetCfg in oracle/detector_ref.cpp"""
    _fields_ = [("mode", _I), ("batch", _I), ("img_h", _I), ("img_w", _I), ("blocks", _I * 4),
                ("num_classes", _I), ("rpn_channels", _I), ("A", _I), ("pool", _I), ("sampling_ratio", _I),
                ("rpn_batch", _I), ("eps", _F), ("slope", _F)]


_REF_SIGS.update({
    "ref_det_param_list": (_I, [_P, _P, _P, _P, _I]),
    "ref_det_step": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _I, _D, _P, _P, _P, _P]),
})

_orc = None
_ref = None


def _load(path, sigs):
    lb = C.CDLL(path)
    for name, (res, args) in sigs.items():
        if not hasattr(lb, name):
            continue
        fn = getattr(lb, name)
        fn.restype = res
        fn.argtypes = args
    return lb


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_PATH):
            raise ImportError(f"{ORC_PATH} missing (make -C oracle)")
        _orc = _load(ORC_PATH, _ORC_SIGS)
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise ImportError(f"{REF_PATH} missing (needs /root/reference to build)")
        _ref = _load(REF_PATH, _REF_SIGS)
    return _ref


def p(a: np.ndarray):
    """ctypes pointer for a C-contiguous numpy array."""
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)
