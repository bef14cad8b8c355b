"""ORACLE — test infrastructure only (never imported by the product package).

ctypes front end over the two CPU checkers that export the C API of
oracle/capi_impl.hpp:

* ``liboracle.so``          this repo's restatement of the reference path
* ``_ref/libouro_ref.so``   the same driver on the reference's own compiled code

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU baseline
load this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libouro_ref.so")
REF_SRC = "/root/reference/proj"

_P = C.c_void_p
_SZ = C.c_size_t
_PD = C.POINTER(C.c_double)


def build(ref: bool | None = None) -> None:
    """Compile liboracle.so (always) and the reference build (when the
    reference sources are present, i.e. in the build container)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"REF={REF_SRC}"], check=True)
        # the C++ host API checked against the reference (needs libouro_b200.so built first)
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_2503_10959_b200", "libouro_b200.so")):
            subprocess.run(["make", "-s", "-C", HERE, "cpp-api-test", f"REF={REF_SRC}"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags.c_contiguous
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class Dims:
    image: int = 32
    channels: int = 3
    patch: int = 4
    embed: int = 16
    state: int = 4
    blocks: int = 2
    classes: int = 10
    conv_width: int = 3

    @property
    def grid(self) -> int:
        return self.image // self.patch

    @property
    def tokens(self) -> int:
        return self.grid * self.grid

    @property
    def pix(self) -> int:
        return self.image * self.image * self.channels

    def as_array(self) -> np.ndarray:
        return np.array([self.image, self.channels, self.patch, self.embed, self.state, self.blocks,
                         self.classes, self.conv_width], dtype=np.uint64)


@dataclass
class Spec:
    wbits: int = 4
    abits: int = 8
    obits: int = 8
    n_refresh: int = 10
    rho: float = 0.01
    d1: bool = True
    d2: bool = True

    def bits(self) -> np.ndarray:
        return np.array([self.wbits, self.abits, self.obits], dtype=np.uint32)


@dataclass
class TensorCal:
    theta: float
    s_in: np.ndarray
    s_full: np.ndarray
    excluded: np.ndarray


@dataclass
class Calibration:
    """Host copy of a calibration: scan tensors [block][dir][kind] and linear
    sites [block][site] (site 0 in_proj, 1..ndirs x_proj, ndirs+1 out_proj)."""
    spec: Spec
    scan: list = field(default_factory=list)
    lin: list = field(default_factory=list)


class OracleError(RuntimeError):
    pass


class Checker:
    def __init__(self, so_path: str = ORACLE_SO):
        if not os.path.exists(so_path):
            raise FileNotFoundError(f"{so_path} not built (run oracle.build())")
        self.path = so_path
        L = self.lib = C.CDLL(so_path)
        L.oro_last_error.restype = C.c_char_p
        L.oro_model_create.argtypes = [_P, _P, _SZ, C.c_uint64, C.POINTER(_P)]
        L.oro_model_free.argtypes = [_P]
        L.oro_model_get.argtypes = [_P, C.c_char_p, _P, _SZ]
        L.oro_model_get.restype = C.c_long
        L.oro_model_set.argtypes = [_P, C.c_char_p, _P, _SZ]
        L.oro_model_qweight.argtypes = [_P, C.c_uint, C.c_char_p, _P, _P, _SZ, _SZ]
        L.oro_model_qweight.restype = C.c_long
        L.oro_normal_fill.argtypes = [C.c_uint64, _P, _SZ]
        L.oro_calibrate.argtypes = [_P, _P, _SZ, _P, _SZ, C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]
        L.oro_calib_new.argtypes = [_P, _P, _SZ, C.c_double, C.c_int, C.c_int, C.POINTER(_P)]
        L.oro_calib_free.argtypes = [_P]
        L.oro_calib_count.argtypes = [_P, C.c_int]
        L.oro_calib_count.restype = C.c_long
        L.oro_calib_get.argtypes = [_P, C.c_int, _SZ, _PD, _P, _P, _P]
        L.oro_calib_set.argtypes = [_P, C.c_int, _SZ, C.c_double, _P, _P, _P]
        L.oro_forward.argtypes = [_P, _P, C.c_int, C.c_int, C.c_int, _P, _SZ, C.c_int, _P]
        L.oro_trace.argtypes = [_P, _P, C.c_int, C.c_int, C.c_int, _P, _SZ, C.POINTER(_P)]
        L.oro_trace_get.argtypes = [_P, C.c_char_p, _P, _SZ]
        L.oro_trace_get.restype = C.c_long
        L.oro_trace_free.argtypes = [_P]
        L.oro_quant_stream.argtypes = [_P, _SZ, _SZ, _SZ, _SZ, C.c_double, _P, _P, _SZ, C.c_uint, C.c_uint,
                                       C.c_int, _P, _P]
        L.oro_hybrid_gemm.argtypes = [_P, _P, _SZ, _SZ, _P, _SZ, C.c_double, _P, _SZ, _P, _P, _P, _P, _P]
        L.oro_split_quantize.argtypes = [_P, _SZ, _SZ, _P, _SZ, C.c_double, C.c_uint, C.c_uint, _P, _P, _P]
        L.oro_pack_int4.argtypes = [_P, _SZ, _SZ, _P]
        if hasattr(L, "ref_pin_fp_forward"):
            L.ref_pin_fp_forward.argtypes = [_P, _P, _SZ, _P]
            L.ref_pin_calibrate.argtypes = [_P, _P, _SZ, _P, _SZ, C.c_double, C.POINTER(_P)]
            L.ref_pin_quantized_forward.argtypes = [_P, _P, C.c_int, _P, _SZ, _P, _P]
            L.ref_pin_save_calibration.argtypes = [_P, C.c_char_p]
            L.ref_pin_quant_eval.argtypes = [_P, _P, C.c_int, _P, _SZ, _P, _P, C.POINTER(C.c_double),
                                             C.POINTER(_SZ), _P]
            L.ref_pin_load_calibration.argtypes = [C.c_char_p, C.POINTER(_P)]
            L.ref_pin_quant_eval_spiked.argtypes = [_P, _P, C.c_int, _P, _SZ, _P, _P, C.POINTER(C.c_double),
                                                    C.POINTER(_SZ), _P, C.c_double, C.c_double, _SZ, C.c_uint64]
            L.ref_pin_refresh_sweep.argtypes = [_P, _SZ, _SZ, _SZ, _SZ, _SZ, _SZ, C.c_double, C.c_double, _SZ,
                                                C.c_uint64, _P, _P]
            L.ref_pin_gemm_bench.argtypes = [_P, _SZ, C.c_double, _SZ, C.c_uint64, _P, _P]
            L.ref_pin_run_id.argtypes = [C.c_char_p, C.c_char_p, _SZ]
            L.ref_pin_run_quant_eval.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p]
            L.ref_pin_run_calib.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p]
            L.ref_pin_write_tensor.argtypes = [C.c_char_p, C.c_int, _P, _SZ, _P]
            L.ref_pin_read_tensor_codes.argtypes = [C.c_char_p, C.c_int, _P, _SZ, C.POINTER(_SZ)]

    def _check(self, st: int) -> None:
        if st != 0:
            raise OracleError(self.lib.oro_last_error().decode())

    # ---- the reference's own pipeline stages and tensor files (reference build only) ----
    def ref_run_id(self, config_text: str) -> str:
        buf = C.create_string_buffer(64)
        self._check(self.lib.ref_pin_run_id(config_text.encode(), buf, 64))
        return buf.value.decode()

    def ref_run_quant_eval(self, config_text: str, calib_dir, images_file, out_dir) -> None:
        self._check(self.lib.ref_pin_run_quant_eval(config_text.encode(), str(calib_dir).encode(),
                                                    str(images_file).encode(), str(out_dir).encode()))

    def ref_run_calib(self, config_text: str, images_file, out_dir) -> None:
        self._check(self.lib.ref_pin_run_calib(config_text.encode(), str(images_file).encode(), str(out_dir).encode()))

    def ref_write_tensor(self, path, dtype: int, data: np.ndarray) -> None:
        """write_tensor_f64 (dtype 0) / _i8 (1) / _u4 (2) of the reference."""
        arr = np.ascontiguousarray(data, np.float64 if dtype == 0 else np.int8)
        shape = np.array(arr.shape, dtype=np.uint64)
        self._check(self.lib.ref_pin_write_tensor(str(path).encode(), dtype, _ptr(shape), arr.ndim, _ptr(arr)))

    def ref_read_tensor_codes(self, path, dtype: int, n: int) -> np.ndarray:
        """read_tensor_i8 (dtype 1) / read_tensor_u4 (2) of the reference (flat codes)."""
        out = np.zeros(max(n, 1), np.int8)
        got = _SZ()
        self._check(self.lib.ref_pin_read_tensor_codes(str(path).encode(), dtype, _ptr(out), out.size, C.byref(got)))
        return out[:got.value]

    # ---- model ---------------------------------------------------------------
    def model(self, dims: Dims, seed: int, orders=(0, 1)) -> "Model":
        h = _P()
        o = np.array(orders, dtype=np.int32)
        self._check(self.lib.oro_model_create(_ptr(dims.as_array()), _ptr(o), len(orders), seed, C.byref(h)))
        return Model(self, h, dims, tuple(orders))

    def normal(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self.lib.oro_normal_fill(seed, _ptr(out), n)
        return out

    # ---- operators -----------------------------------------------------------
    def quant_stream(self, x: np.ndarray, theta: float, s_in: np.ndarray, s_full: np.ndarray, n_refresh: int,
                     abits: int, obits: int, mode: int = 1):
        """x: [S][T][E][N] f64 (copied). Returns (x_fq, masks[S,T,E], scanned[S,T])."""
        x = np.ascontiguousarray(x, dtype=np.float64).copy()
        S, T, E, N = x.shape
        masks = np.zeros((S, T, E), dtype=np.uint8)
        scanned = np.zeros((S, T), dtype=np.uint8)
        self._check(self.lib.oro_quant_stream(_ptr(x), S, T, E, N, theta, _ptr(np.ascontiguousarray(s_in, np.float64)),
                                              _ptr(np.ascontiguousarray(s_full, np.float64)), n_refresh, abits, obits,
                                              mode, _ptr(masks), _ptr(scanned)))
        return x, masks, scanned

    def ref_refresh_sweep(self, periods, steps, m, k, c, persistent, transient_rate, spike_gain, trials, seed):
        """The reference's own bench_refresh_sweep (gemm.cpp:326-411): (mean_o_list, scans_per_step) per period."""
        per = np.ascontiguousarray(periods, np.uint64)
        mo = np.zeros(len(per))
        sc = np.zeros(len(per))
        self._check(self.lib.ref_pin_refresh_sweep(_ptr(per), len(per), steps, m, k, c, persistent, transient_rate,
                                                   spike_gain, trials, seed, _ptr(mo), _ptr(sc)))
        return mo, sc

    def ref_gemm_bench(self, sizes, outlier_fraction, trials, seed):
        """The reference's own bench_gemm (gemm.cpp:260-324): its (path, size) record list."""
        sz = np.ascontiguousarray(sizes, np.uint64)
        paths = np.zeros(2 * len(sz), np.int32)
        out = np.zeros(2 * len(sz), np.uint64)
        self._check(self.lib.ref_pin_gemm_bench(_ptr(sz), len(sz), outlier_fraction, trials, seed, _ptr(paths),
                                                _ptr(out)))
        return list(zip(paths.tolist(), out.tolist()))

    def hybrid_gemm(self, w: np.ndarray, w_scales: np.ndarray, x_inlier: np.ndarray, s_in: float,
                    channels: np.ndarray, ocodes: np.ndarray, oscales: np.ndarray):
        w = np.ascontiguousarray(w, np.int8)
        m, k = w.shape
        x_inlier = np.ascontiguousarray(x_inlier, np.int8)
        c = x_inlier.shape[1]
        ch = np.ascontiguousarray(channels, np.uint64)
        oc = np.ascontiguousarray(ocodes, np.int8).reshape(len(ch), c) if len(ch) else np.zeros((0, c), np.int8)
        os_ = np.ascontiguousarray(oscales, np.float64)
        acc_in = np.zeros((m, c), np.int32)
        acc_out = np.zeros((m, c), np.int32)
        out = np.zeros((m, c), np.float64)
        self._check(self.lib.oro_hybrid_gemm(_ptr(w), _ptr(np.ascontiguousarray(w_scales, np.float64)), m, k,
                                             _ptr(x_inlier), c, s_in, _ptr(ch), len(ch), _ptr(oc), _ptr(os_),
                                             _ptr(acc_in), _ptr(acc_out), _ptr(out)))
        return acc_in, acc_out, out

    def split_quantize(self, x: np.ndarray, channels, s_in: float, abits: int, obits: int):
        x = np.ascontiguousarray(x, np.float64)
        k, c = x.shape
        ch = np.ascontiguousarray(channels, np.uint64)
        inl = np.zeros((k, c), np.int8)
        oc = np.zeros((max(len(ch), 1), c), np.int8)
        os_ = np.zeros(max(len(ch), 1), np.float64)
        self._check(self.lib.oro_split_quantize(_ptr(x), k, c, _ptr(ch), len(ch), s_in, abits, obits, _ptr(inl),
                                                _ptr(oc), _ptr(os_)))
        return inl, oc[:len(ch)], os_[:len(ch)]

    def pack_int4(self, codes: np.ndarray) -> np.ndarray:
        codes = np.ascontiguousarray(codes, np.int8)
        r, c = codes.shape
        out = np.zeros((r, (c + 1) // 2), np.uint8)
        self._check(self.lib.oro_pack_int4(_ptr(codes), r, c, _ptr(out)))
        return out


class Model:
    def __init__(self, chk: Checker, h, dims: Dims, orders):
        self.chk, self.h, self.dims, self.orders = chk, h, dims, orders

    def __del__(self):
        try:
            self.chk.lib.oro_model_free(self.h)
        except Exception:
            pass

    def get(self, name: str) -> np.ndarray:
        n = self.chk.lib.oro_model_get(self.h, name.encode(), None, 0)
        if n < 0:
            raise KeyError(name)
        out = np.empty(n, np.float64)
        self.chk.lib.oro_model_get(self.h, name.encode(), _ptr(out), n)
        return out

    def set(self, name: str, v: np.ndarray) -> None:
        v = np.ascontiguousarray(v, np.float64).ravel()
        self.chk._check(self.chk.lib.oro_model_set(self.h, name.encode(), _ptr(v), v.size))

    def tensor_names(self):
        names = ["patch_w", "patch_b", "head_w", "head_b"]
        for b in range(self.dims.blocks):
            names += [f"block{b}.{f}" for f in ("w_in", "w_gate", "conv", "out_proj")]
            for d in range(len(self.orders)):
                names += [f"block{b}.dir{d}.{f}" for f in ("a", "w_b", "w_c", "w_delta", "b_delta")]
        return names

    def qweight(self, which: str, bits: int = 4):
        n = self.chk.lib.oro_model_qweight(self.h, bits, which.encode(), None, None, 0, 0)
        if n < 0:
            raise OracleError(self.chk.lib.oro_last_error().decode())
        codes = np.empty(n, np.int8)
        scales = np.empty(n, np.float64)
        self.chk.lib.oro_model_qweight(self.h, bits, which.encode(), _ptr(codes), _ptr(scales), n, n)
        return codes, scales

    def calibrate(self, images: np.ndarray, spec: Spec, threads: int = 8) -> "CalibHandle":
        images = np.ascontiguousarray(images, np.float64)
        B = images.size // self.dims.pix
        h = _P()
        self.chk._check(self.chk.lib.oro_calibrate(self.h, _ptr(images), B, _ptr(spec.bits()), spec.n_refresh,
                                                   spec.rho, int(spec.d1), int(spec.d2), threads, C.byref(h)))
        return CalibHandle(self, h, spec)

    def calib_from(self, cal: Calibration) -> "CalibHandle":
        h = _P()
        s = cal.spec
        self.chk._check(self.chk.lib.oro_calib_new(self.h, _ptr(s.bits()), s.n_refresh, s.rho, int(s.d1), int(s.d2),
                                                   C.byref(h)))
        ch = CalibHandle(self, h, s)
        for which, lst in ((0, cal.scan), (1, cal.lin)):
            for i, t in enumerate(lst):
                self.chk._check(self.chk.lib.oro_calib_set(
                    h, which, i, t.theta, _ptr(np.ascontiguousarray(t.s_in, np.float64)),
                    _ptr(np.ascontiguousarray(t.s_full, np.float64)),
                    _ptr(np.ascontiguousarray(t.excluded, np.uint8))))
        return ch

    def forward(self, images: np.ndarray, calib: "CalibHandle | None", mode: int, d1: bool = True, d2: bool = True,
                threads: int = 8) -> np.ndarray:
        images = np.ascontiguousarray(images, np.float64)
        B = images.size // self.dims.pix
        logits = np.zeros((B, self.dims.classes), np.float64)
        self.chk._check(self.chk.lib.oro_forward(self.h, calib.h if calib else None, mode, int(d1), int(d2),
                                                 _ptr(images), B, threads, _ptr(logits)))
        return logits

    def trace(self, image: np.ndarray, calib: "CalibHandle | None", mode: int, block: int, d1: bool = True,
              d2: bool = True) -> "Trace":
        image = np.ascontiguousarray(image, np.float64)
        h = _P()
        self.chk._check(self.chk.lib.oro_trace(self.h, calib.h if calib else None, mode, int(d1), int(d2),
                                               _ptr(image), block, C.byref(h)))
        return Trace(self.chk, h)

    # reference-only pins
    def ref_fp_forward(self, images: np.ndarray) -> np.ndarray:
        images = np.ascontiguousarray(images, np.float64)
        B = images.size // self.dims.pix
        logits = np.zeros((B, self.dims.classes), np.float64)
        self.chk._check(self.chk.lib.ref_pin_fp_forward(self.h, _ptr(images), B, _ptr(logits)))
        return logits

    def ref_calibrate(self, images: np.ndarray, spec: Spec) -> "CalibHandle":
        images = np.ascontiguousarray(images, np.float64)
        B = images.size // self.dims.pix
        h = _P()
        self.chk._check(self.chk.lib.ref_pin_calibrate(self.h, _ptr(images), B, _ptr(spec.bits()), spec.n_refresh,
                                                       spec.rho, C.byref(h)))
        return CalibHandle(self, h, Spec(spec.wbits, spec.abits, spec.obits, spec.n_refresh, spec.rho, False, False))

    def ref_quantized_forward(self, images: np.ndarray, calib: "CalibHandle", mode: int):
        images = np.ascontiguousarray(images, np.float64)
        B = images.size // self.dims.pix
        lq = np.zeros((B, self.dims.classes), np.float64)
        lf = np.zeros((B, self.dims.classes), np.float64)
        self.chk._check(self.chk.lib.ref_pin_quantized_forward(self.h, calib.h, mode, _ptr(images), B, _ptr(lq),
                                                               _ptr(lf)))
        return lq, lf

    def ref_quant_eval(self, images: np.ndarray, calib: "CalibHandle", mode: int, spikes=None) -> dict:
        """The reference's quantized_forward (quant.cpp:505-579) and its metrics;
        spikes = (rate, gain, channels, salt) for its SpikeSettings."""
        images = np.ascontiguousarray(images, np.float64)
        B = images.size // self.dims.pix
        lq = np.zeros((B, self.dims.classes), np.float64)
        lf = np.zeros((B, self.dims.classes), np.float64)
        mse, agree = C.c_double(), _SZ()
        lm = np.zeros(self.dims.blocks * len(self.orders), np.float64)
        if spikes is not None:
            self.chk._check(self.chk.lib.ref_pin_quant_eval_spiked(self.h, calib.h, mode, _ptr(images), B, _ptr(lq),
                                                                   _ptr(lf), C.byref(mse), C.byref(agree), _ptr(lm),
                                                                   *spikes))
        else:
            self.chk._check(self.chk.lib.ref_pin_quant_eval(self.h, calib.h, mode, _ptr(images), B, _ptr(lq),
                                                            _ptr(lf), C.byref(mse), C.byref(agree), _ptr(lm)))
        return dict(logits_q=lq, logits_fp=lf, logits_mse=mse.value, argmax_agree=agree.value, layer_mse=lm)

    def ref_save_calibration(self, calib: "CalibHandle", directory: str) -> None:
        """The reference's own save_calibration (quant.cpp:179-216) of a handle's scan tensors."""
        self.chk._check(self.chk.lib.ref_pin_save_calibration(calib.h, str(directory).encode()))

    def ref_load_calibration(self, directory: str, spec: Spec) -> "CalibHandle":
        """The reference's own load_calibration (quant.cpp:218-290)."""
        h = C.c_void_p()
        self.chk._check(self.chk.lib.ref_pin_load_calibration(str(directory).encode(), C.byref(h)))
        return CalibHandle(self, h, spec)


class CalibHandle:
    def __init__(self, model: Model, h, spec: Spec):
        self.model, self.h, self.spec = model, h, spec

    def __del__(self):
        try:
            self.model.chk.lib.oro_calib_free(self.h)
        except Exception:
            pass

    def export(self) -> Calibration:
        lib = self.model.chk.lib
        L, E = self.model.dims.tokens, self.model.dims.embed
        cal = Calibration(self.spec)
        for which, lst in ((0, cal.scan), (1, cal.lin)):
            for i in range(lib.oro_calib_count(self.h, which)):
                th = C.c_double()
                si = np.empty(L, np.float64)
                sf = np.empty(L, np.float64)
                ex = np.empty(E, np.uint8)
                self.model.chk._check(lib.oro_calib_get(self.h, which, i, C.byref(th), _ptr(si), _ptr(sf), _ptr(ex)))
                lst.append(TensorCal(th.value, si, sf, ex))
        return cal


class Trace:
    DT = {"codes": np.int8, "ocode": np.int8, "omask": np.uint8, "oscale": np.float64, "acc_in": np.int32,
          "acc_out": np.int32, "out": np.float64, "scanned": np.uint8}

    def __init__(self, chk: Checker, h):
        self.chk, self.h = chk, h

    def __del__(self):
        try:
            self.chk.lib.oro_trace_free(self.h)
        except Exception:
            pass

    def get(self, key: str) -> np.ndarray:
        n = self.chk.lib.oro_trace_get(self.h, key.encode(), None, 0)
        if n < 0:
            raise KeyError(key)
        leaf = key.split(".")[-1]
        dt = self.DT.get(leaf, np.float64)
        if leaf.startswith("mask") or leaf.startswith("scanned"):
            dt = np.uint8
        out = np.empty(n // np.dtype(dt).itemsize, dt)
        self.chk.lib.oro_trace_get(self.h, key.encode(), _ptr(out), n)
        return out
