"""Host-side objects over the C ABI: Context (device + stream), Model (weights
resident in HBM), Calibration (CalibrationResult + D2 sites) and the operator
entry points (K1 detect/quantize, K2 quant-linear, K3 quantized scan, f64
projection). Device buffers are torch CUDA tensors; only their pointers cross
the boundary.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


def _ptr(t):
    """Raw pointer of a torch tensor / numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        assert t.flags.c_contiguous
        return t.ctypes.data_as(C.c_void_p)
    assert t.is_contiguous(), "tensors crossing the C ABI must be contiguous"
    return C.c_void_p(t.data_ptr())


@dataclass
class Dims:
    """ModelDims (ssm.hpp:42-56)."""
    image: int = 224
    channels: int = 3
    patch: int = 16
    embed: int = 768
    state: int = 16
    blocks: int = 24
    classes: int = 1000
    conv_width: int = 4

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
        return np.array([self.image, self.channels, self.patch, self.embed, self.state, self.blocks, self.classes,
                         self.conv_width], dtype=np.uint64)


VIM_T = Dims(embed=192)
VIM_S = Dims(embed=384)
VIM_B = Dims(embed=768)


@dataclass
class QuantSpec:
    """QuantSpec (quant.hpp:21-28) + the two declared extensions."""
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


class Context:
    """One device + one stream (ouro_b200_ctx)."""

    def __init__(self, device: int = 0, stream=None):
        """Bind to `stream` (torch.cuda.Stream / raw handle); default: torch's
        current stream, so operator calls are ordered with the torch ops that
        allocate and fill their buffers."""
        self.lib = L.load()
        h = C.c_void_p()
        L.check(self.lib.ouro_b200_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(device)
        self.set_stream(stream)

    def __del__(self):
        try:
            self.lib.ouro_b200_ctx_free(self.h)
        except Exception:
            pass

    def set_stream(self, stream) -> None:
        """Run on a caller stream (torch.cuda.Stream or raw handle)."""
        raw = getattr(stream, "cuda_stream", stream)
        L.check(self.lib.ouro_b200_ctx_set_stream(self.h, C.c_void_p(raw)))

    def synchronize(self) -> None:
        L.check(self.lib.ouro_b200_ctx_synchronize(self.h))

    @property
    def num_sms(self) -> int:
        v = C.c_int()
        L.check(self.lib.ouro_b200_ctx_num_sms(self.h, C.byref(v)))
        return v.value

    def measure_fp64_peak(self) -> float:
        """Measured DFMA throughput of this device in TFLOP/s."""
        v = C.c_double()
        L.check(self.lib.ouro_b200_measure_fp64_peak(self.h, C.byref(v)))
        return v.value

    def measure_i8_peak(self) -> float:
        """Measured dense int8 tensor-core throughput of this device in TOP/s."""
        v = C.c_double()
        L.check(self.lib.ouro_b200_measure_i8_peak(self.h, C.byref(v)))
        return v.value

    def launch_count(self) -> int:
        """Kernels this library launched from the calling thread so far (graph replays excluded)."""
        v = C.c_longlong()
        L.check(self.lib.ouro_b200_launch_count(C.byref(v)))
        return v.value

    def math_eval(self, fn: str, x):
        """Device exp / log1p / softplus / silu of a float64 CUDA tensor: the forms the
        kernels use, which restate glibc's so they equal the reference's bit for bit."""
        code = {"exp": 0, "log1p": 1, "softplus": 2, "silu": 3}[fn]
        x = x.contiguous()
        y = x.new_empty(x.shape)
        L.check(self.lib.ouro_b200_math_eval(self.h, code, _ptr(x), _ptr(y), x.numel()))
        return y

    def refresh_sweep(self, periods=(1, 5, 10, 20, 0), *, steps=300, m=8, k=512, c=32, persistent_channels=6,
                      transient_rate=0.15, spike_gain=40.0, trials=5, seed=1, outputs=False):
        """bench_refresh_sweep (gemm.cpp:326-411) on the GPU: one record per period
        (period, median_total_ns, mean_o_list, scans_per_step); with outputs=True also
        the GEMM outputs [n_periods][steps][c][m]."""
        per = (C.c_size_t * len(periods))(*periods)
        st = L.SweepSettings(per, len(periods), steps, m, k, c, persistent_channels, transient_rate, spike_gain,
                             trials, seed)
        recs = (L.SweepRecord * len(periods))()
        y = np.zeros((len(periods), steps, c, m)) if outputs else None
        L.check(self.lib.ouro_b200_refresh_sweep(self.h, C.byref(st), recs, _ptr(y)))
        out = [dict(period=r.period, median_total_ns=r.median_total_ns, mean_o_list=r.mean_o_list,
                    scans_per_step=r.scans_per_step) for r in recs]
        return (out, y) if outputs else out

    def gemm_bench(self, sizes=(64, 128, 256), *, outlier_fraction=0.01, trials=5, seed=1, f16_output=False):
        """bench_gemm (gemm.cpp:260-324) on the GPU: per size a "hybrid" (K2) and an
        "f64" record with the median device time in ns."""
        sz = (C.c_size_t * len(sizes))(*sizes)
        st = L.BenchSettings(sz, len(sizes), outlier_fraction, trials, seed, int(f16_output))
        recs = (L.BenchRecord * (2 * len(sizes)))()
        L.check(self.lib.ouro_b200_gemm_bench(self.h, C.byref(st), recs))
        return [dict(path="hybrid" if r.path == 0 else "f64", size=r.size, median_ns=r.median_ns) for r in recs]

    def detect_quantize_planes(self, x, *, theta, s_in, n_refresh, act_bits=4, outlier_bits=8, Kp=None):
        """detect_outliers + split_quantize over a stream of K x C planes (x: float64
        CUDA tensor [steps][K][C]) into the K2 operand with rows t*C + i; returns the
        QAct dict plus `scanned` [steps]."""
        import torch
        x, s_in = x.contiguous(), s_in.contiguous()  # kept alive until the call returns
        steps, K, Cc = x.shape
        Kp = K if Kp is None else Kp
        rows, J, dev = steps * Cc, (Kp + 31) // 32, x.device
        out = dict(codes=torch.empty(rows, Kp, dtype=torch.int8, device=dev),
                   s_row=torch.empty(rows, dtype=torch.float64, device=dev),
                   ocnt=torch.empty(rows, dtype=torch.int32, device=dev),
                   omask=torch.zeros(rows, J, dtype=torch.int32, device=dev),
                   ocode=torch.zeros(rows, Kp, dtype=torch.int8, device=dev),
                   oscale=torch.zeros(rows, Kp, dtype=torch.float64, device=dev),
                   scanned=torch.zeros(steps, dtype=torch.uint8, device=dev))
        L.check(self.lib.ouro_b200_detect_quantize_planes(
            self.h, _ptr(x), steps, K, Cc, float(theta), _ptr(s_in), n_refresh, act_bits,
            outlier_bits, Kp, _ptr(out["codes"]), _ptr(out["s_row"]), _ptr(out["ocnt"]), _ptr(out["omask"]),
            _ptr(out["ocode"]), _ptr(out["oscale"]), _ptr(out["scanned"])))
        return out

    # ---- operators (device tensors) --------------------------------------------
    def detect_quantize(self, x, *, S, T, E, theta, s_in, s_full, n_refresh, act_bits, outlier_bits,
                        mode=L.MODE_DYNAMIC, src=L.SRC_PLAIN, x2=None, gate=None, order=-1, grid=0, literal=False,
                        scanned=None, packed=False):
        """K1 over S x T planes. Returns the QAct operand as a dict of device
        tensors: codes (or, packed=True with act_bits 4, codes4: the nibble-packed
        codes [rows][E/2] in pack_int4's layout), s_row, ocnt, omask (uint32 words),
        ocode/oscale (dense, valid at outlier positions)."""
        import torch
        dev = x.device
        rows = S * T
        J = (E + 31) // 32
        s_row = torch.empty(rows, dtype=torch.float64, device=dev)
        ocnt = torch.empty(rows, dtype=torch.int32, device=dev)
        omask = torch.zeros(rows, J, dtype=torch.int32, device=dev)
        ocode = torch.zeros(rows, E, dtype=torch.int8, device=dev)
        oscale = torch.zeros(rows, E, dtype=torch.float64, device=dev)
        if packed:
            if act_bits != 4:
                raise L.ValidationError(2, "detect_quantize: packed codes are 4-bit (act_bits must be 4)")
            codes4 = torch.empty(rows, (E + 1) // 2, dtype=torch.uint8, device=dev)
            L.check(self.lib.ouro_b200_detect_quantize_packed(
                self.h, _ptr(x), _ptr(x2), _ptr(gate), S, T, E, src, order, grid, float(theta), _ptr(s_in),
                _ptr(s_full), n_refresh, outlier_bits, mode, int(literal), _ptr(codes4), _ptr(s_row), _ptr(ocnt),
                _ptr(omask), _ptr(ocode), _ptr(oscale), _ptr(scanned)))
            return dict(codes4=codes4, s_row=s_row, ocnt=ocnt, omask=omask, ocode=ocode, oscale=oscale)
        codes = torch.empty(rows, E, dtype=torch.int8, device=dev)
        L.check(self.lib.ouro_b200_detect_quantize(
            self.h, _ptr(x), _ptr(x2), _ptr(gate), S, T, E, src, order, grid, float(theta), _ptr(s_in), _ptr(s_full),
            n_refresh, act_bits, outlier_bits, mode, int(literal), _ptr(codes), _ptr(s_row), _ptr(ocnt), _ptr(omask),
            _ptr(ocode), _ptr(oscale), _ptr(scanned), None))
        return dict(codes=codes, s_row=s_row, ocnt=ocnt, omask=omask, ocode=ocode, oscale=oscale)

    def quant_linear(self, act: dict, w, wt, ws, *, post=L.POST_STORE, out=None, out2=None, split=0, acc_in=None,
                     acc_out=None, bias=None):
        """K2: hybrid quant-linear over K1's operand dict (int8 `codes` or nibble-packed
        `codes4`); returns `out`."""
        import torch
        packed = "codes4" in act
        M, K = (act["codes4"].shape[0], 2 * act["codes4"].shape[1]) if packed else act["codes"].shape
        R = w.shape[0]
        if out is None:
            out = torch.empty(M, R, dtype=torch.float64, device=w.device)
        ld = out.shape[1]
        fn = self.lib.ouro_b200_quant_linear_packed if packed else self.lib.ouro_b200_quant_linear
        L.check(fn(self.h, M, R, K, _ptr(act["codes4"] if packed else act["codes"]), _ptr(act["s_row"]),
                   _ptr(act["ocnt"]), _ptr(act["omask"]), _ptr(act["ocode"]), _ptr(act["oscale"]), _ptr(w), _ptr(wt),
                   _ptr(ws), post, _ptr(out), ld, _ptr(out2), split, _ptr(bias), _ptr(acc_in), _ptr(acc_out)))
        return out

    def quant_scan(self, *, S, T, E, order, grid, u, proj, a, b_delta, o, mode, n_refresh=10, act_bits=8,
                   outlier_bits=8, theta=None, s_in=None, s_full=None, literal=None, force_literal=False,
                   masks=None, spikes: "SpikeSettings | None" = None, block=0, dir=0, sample0=0):
        """K3 for one direction. theta: 3 floats; s_in/s_full: 3 device tensors each.
        spikes: SpikeHook settings, placed at (sample0 + s, block, dir, t)."""
        th = (C.c_double * 3)(*(theta or (0.0, 0.0, 0.0)))
        si = (C.c_void_p * 3)(*[t.data_ptr() for t in s_in]) if s_in is not None else None
        sf = (C.c_void_p * 3)(*[t.data_ptr() for t in s_full]) if s_full is not None else None
        if spikes is not None:
            sp = L.Spikes(spikes.rate, spikes.gain, spikes.channels, spikes.salt, spikes.sample0)
            L.check(self.lib.ouro_b200_quant_scan_spiked(
                self.h, S, T, E, 16, order, grid, _ptr(u), _ptr(proj), _ptr(a), _ptr(b_delta), _ptr(o), mode,
                n_refresh, act_bits, outlier_bits, th if theta is not None else None, si, sf, C.byref(sp), block, dir,
                sample0))
            return o
        L.check(self.lib.ouro_b200_quant_scan(
            self.h, S, T, E, 16, order, grid, _ptr(u), _ptr(proj), _ptr(a), _ptr(b_delta), _ptr(o), mode, n_refresh,
            act_bits, outlier_bits, th if theta is not None else None, si, sf, _ptr(literal), int(force_literal),
            _ptr(masks)))
        return o

    def dgemm(self, a, w, *, post=L.POST_STORE, out=None, out2=None, split=0, bias=None):
        import torch
        M, K = a.shape
        R = w.shape[0]
        if out is None:
            out = torch.empty(M, R, dtype=torch.float64, device=a.device)
        L.check(self.lib.ouro_b200_dgemm(self.h, M, R, K, _ptr(a), a.stride(0), _ptr(w), post, _ptr(out),
                                         out.shape[1], _ptr(out2), split, _ptr(bias)))
        return out


@dataclasses.dataclass
class SpikeSettings:
    """SpikeSettings (quant.hpp:105-110): per (sample, block, dir, step) probability
    `rate` of multiplying `channels` hashed channels' b_bar by `gain`."""
    rate: float = 0.0
    gain: float = 100.0
    channels: int = 1
    salt: int = 0
    sample0: int = 0  # global index of the call's first sample (a batch sharded across GPUs)


class Calibration:
    """CalibrationResult (quant.hpp:44-49): scan tensors [block][dir][kind]
    plus (D2) linear-input sites [block][site]."""

    def __init__(self, model: "Model", h, spec: QuantSpec):
        self.model, self.h, self.spec = model, h, spec
        self.lib = model.lib

    def __del__(self):
        try:
            self.lib.ouro_b200_calib_free(self.h)
        except Exception:
            pass

    def count(self, which: int) -> int:
        n = C.c_size_t()
        L.check(self.lib.ouro_b200_calib_count(self.h, which, C.byref(n)))
        return n.value

    def get(self, which: int, idx: int) -> TensorCal:
        d = self.model.dims
        th = C.c_double()
        si = np.empty(d.tokens, np.float64)
        sf = np.empty(d.tokens, np.float64)
        ex = np.empty(d.embed, np.uint8)
        L.check(self.lib.ouro_b200_calib_get(self.h, which, idx, C.byref(th), _ptr(si), _ptr(sf), _ptr(ex)))
        return TensorCal(th.value, si, sf, ex)

    def set(self, which: int, idx: int, tc: TensorCal) -> None:
        L.check(self.lib.ouro_b200_calib_set(self.h, which, idx, float(tc.theta),
                                             _ptr(np.ascontiguousarray(tc.s_in, np.float64)),
                                             _ptr(np.ascontiguousarray(tc.s_full, np.float64)),
                                             _ptr(np.ascontiguousarray(tc.excluded, np.uint8))))

    def export(self):
        return ([self.get(0, i) for i in range(self.count(0))], [self.get(1, i) for i in range(self.count(1))])

    def save(self, directory: str) -> None:
        """Write the reference's calibration directory (save_calibration,
        quant.cpp:179-216) plus the D2 linear-site tables (d2_linear_sites.txt)."""
        L.check(self.lib.ouro_b200_calib_save(self.h, self.model.h, str(directory).encode()))


class Trace:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            self.lib.ouro_b200_trace_free(self.h)
        except Exception:
            pass

    def get(self, key: str, dtype) -> np.ndarray:
        n = C.c_size_t()
        L.check(self.lib.ouro_b200_trace_get(self.h, key.encode(), None, 0, C.byref(n)))
        out = np.empty(n.value // np.dtype(dtype).itemsize, dtype)
        L.check(self.lib.ouro_b200_trace_get(self.h, key.encode(), _ptr(out), n.value, C.byref(n)))
        return out

    def has(self, key: str) -> bool:
        n = C.c_size_t()
        return self.lib.ouro_b200_trace_get(self.h, key.encode(), None, 0, C.byref(n)) == 0


def _scan_perm(order: int, T: int, grid: int) -> np.ndarray:
    """scan_permutation (ssm.cpp:30-46): canonical token visited at scan step t."""
    t = np.arange(T)
    fast, slow = t % grid, t // grid
    return {0: slow * grid + fast, 1: T - 1 - (slow * grid + fast), 2: fast * grid + slow,
            3: T - 1 - (fast * grid + slow)}[order]


class Model:
    """Toy Vim model (ToyVmmModel, ssm.hpp:58-66) resident on one B200."""

    def __init__(self, ctx: Context, dims: Dims, seed: int, orders=(0, 1)):
        self.ctx, self.lib, self.dims, self.orders = ctx, ctx.lib, dims, tuple(orders)
        h = C.c_void_p()
        o = np.array(orders, dtype=np.int32)
        L.check(self.lib.ouro_b200_model_create(ctx.h, _ptr(dims.as_array()), _ptr(o), len(orders), seed,
                                                C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.lib.ouro_b200_model_free(self.h)
        except Exception:
            pass

    def set_tensor(self, name: str, v: np.ndarray) -> None:
        v = np.ascontiguousarray(v, np.float64).ravel()
        L.check(self.lib.ouro_b200_model_set_tensor(self.h, name.encode(), _ptr(v), v.size))

    def get_tensor(self, name: str) -> np.ndarray:
        n = C.c_size_t()
        L.check(self.lib.ouro_b200_model_get_tensor(self.h, name.encode(), None, 0, C.byref(n)))
        out = np.empty(n.value, np.float64)
        L.check(self.lib.ouro_b200_model_get_tensor(self.h, name.encode(), _ptr(out), n.value, C.byref(n)))
        return out

    def new_calibration(self, spec: QuantSpec) -> Calibration:
        h = C.c_void_p()
        L.check(self.lib.ouro_b200_calib_create(self.h, _ptr(spec.bits()), spec.n_refresh, spec.rho, int(spec.d1),
                                                int(spec.d2), C.byref(h)))
        return Calibration(self, h, spec)

    def calibration_from(self, scan, lin, spec: QuantSpec) -> Calibration:
        cal = self.new_calibration(spec)
        for i, t in enumerate(scan):
            cal.set(0, i, t)
        for i, t in enumerate(lin):
            cal.set(1, i, t)
        return cal

    def load_calibration(self, directory: str, d1: bool = True, d2: bool = True) -> Calibration:
        """Read a calibration directory (load_calibration, quant.cpp:218-290);
        d2 needs the D2 tables this library writes (reference-written: d2=False)."""
        h = C.c_void_p()
        L.check(self.lib.ouro_b200_calib_load(self.h, str(directory).encode(), int(d1), int(d2), C.byref(h)))
        bits = (C.c_uint * 3)()
        nr, rho, k1, k2 = C.c_size_t(), C.c_double(), C.c_int(), C.c_int()
        L.check(self.lib.ouro_b200_calib_spec(h, bits, C.byref(nr), C.byref(rho), C.byref(k1), C.byref(k2)))
        spec = QuantSpec(int(bits[0]), int(bits[1]), int(bits[2]), int(nr.value), float(rho.value), bool(k1.value),
                         bool(k2.value))
        return Calibration(self, h, spec)

    def calibrate(self, images, spec: QuantSpec, chunk: int = 0) -> Calibration:
        """calibrate (quant.cpp:129-177) on the GPU; images: device f64 tensor [B, H, W, C]."""
        h = C.c_void_p()
        B = images.numel() // self.dims.pix
        L.check(self.lib.ouro_b200_calibrate(self.h, _ptr(images), B, _ptr(spec.bits()), spec.n_refresh, spec.rho,
                                             int(spec.d1), int(spec.d2), chunk, C.byref(h)))
        return Calibration(self, h, spec)

    def set_option(self, key: str, value: int) -> None:
        """Engine option, e.g. scan_variant (0 auto, 1 reference kernel, 2 exact codes, 3 / 6 two threads per
        channel with the f32 / f64 state update, 4 / 5 one thread per channel with the f64 / f32 state update, 7 the
        one-thread f32-state kernel in its large-grid shape)."""
        L.check(self.lib.ouro_b200_model_set_option(self.h, key.encode(), int(value)))

    def use_graphs(self, on: bool = True) -> None:
        L.check(self.lib.ouro_b200_model_use_graphs(self.h, int(on)))

    def forward(self, images, calib: Calibration | None, mode: int, *, d1=True, d2=True, logits=None):
        """Device forward: images f64 CUDA tensor [B, H, W, C] -> logits f64 [B, classes] (async)."""
        import torch
        B = images.numel() // self.dims.pix
        if logits is None:
            logits = torch.empty(B, self.dims.classes, dtype=torch.float64, device=images.device)
        L.check(self.lib.ouro_b200_forward(self.h, calib.h if calib else None, mode, int(d1), int(d2),
                                           _ptr(images), B, _ptr(logits)))
        return logits

    FAMILIES = ("k1_detect_quant", "k2_quant_linear", "k3_scan", "f64_projection", "aux")

    def forward_profile(self, images, calib, mode: int, *, d1=True, d2=True, logits=None):
        """One forward with per-kernel-family CUDA-event timing -> (logits, {family: (ms, launches)})."""
        import torch
        B = images.numel() // self.dims.pix
        if logits is None:
            logits = torch.empty(B, self.dims.classes, dtype=torch.float64, device=images.device)
        ms = (C.c_double * 5)()
        n = (C.c_int * 5)()
        L.check(self.lib.ouro_b200_forward_profile(self.h, calib.h if calib else None, mode, int(d1), int(d2),
                                                   _ptr(images), B, _ptr(logits), ms, n))
        return logits, {f: (ms[i], n[i]) for i, f in enumerate(self.FAMILIES)}

    def forward_profile_launches(self, images, calib, mode: int, *, d1=True, d2=True, logits=None):
        """One forward with CUDA events around every launch -> [(family, ms)] in issue order."""
        import torch
        B = images.numel() // self.dims.pix
        if logits is None:
            logits = torch.empty(B, self.dims.classes, dtype=torch.float64, device=images.device)
        cap = 4096
        ms = (C.c_double * cap)()
        fam = (C.c_int * cap)()
        n = C.c_size_t()
        L.check(self.lib.ouro_b200_forward_profile_launches(self.h, calib.h if calib else None, mode, int(d1),
                                                            int(d2), _ptr(images), B, _ptr(logits), ms, fam, cap,
                                                            C.byref(n)))
        return [(self.FAMILIES[fam[k]], ms[k]) for k in range(min(n.value, cap))]

    def forward_host(self, images: np.ndarray, calib: Calibration | None, mode: int, *, d1=True, d2=True,
                     logits: np.ndarray | None = None) -> np.ndarray:
        """End-to-end call with host buffers (H2D + forward + D2H inside)."""
        images = np.ascontiguousarray(images, np.float64)
        B = images.size // self.dims.pix
        if logits is None:
            logits = np.empty((B, self.dims.classes), np.float64)
        L.check(self.lib.ouro_b200_forward_host(self.h, calib.h if calib else None, mode, int(d1), int(d2),
                                                _ptr(images), B, _ptr(logits)))
        return logits

    def qweight(self, name: str, bits: int = 4) -> np.ndarray:
        """W4 dequantized operand (quantize_weights + dequantize_rows, quant.cpp:355-384):
        patch_w, head_w, block<b>.in, block<b>.out_proj, block<b>.conv, block<b>.dir<d>.xp."""
        n = C.c_size_t()
        L.check(self.lib.ouro_b200_model_get_qweight(self.h, name.encode(), bits, None, 0, C.byref(n)))
        out = np.empty(n.value, np.float64)
        L.check(self.lib.ouro_b200_model_get_qweight(self.h, name.encode(), bits, _ptr(out), n.value, C.byref(n)))
        return out

    def set_spikes(self, spikes: "SpikeSettings | None") -> None:
        """SpikeHook for every later forward / trace (None or rate 0 = off)."""
        sp = L.Spikes(spikes.rate, spikes.gain, spikes.channels, spikes.salt, spikes.sample0) if spikes is not None else None
        L.check(self.lib.ouro_b200_model_set_spikes(self.h, C.byref(sp) if sp is not None else None))

    def quant_eval(self, images: np.ndarray, calib: Calibration, mode: int, *, d1=True, d2=True,
                   spikes: "SpikeSettings | None" = None) -> dict:
        """quantized_forward (quant.cpp:505-579) on the GPU: the FP pass and the
        quantized pass over host images, logits_mse over all logits, argmax
        agreement, and the teacher-forced scan-output MSE per (block, dir) -- each
        direction's quantized scan re-run on the FP pass's own scan input with the
        W4 x_proj weights (quant.cpp:548-577). spikes: the SpikeHook of all three
        passes (rate 0 / None = off)."""
        if spikes is not None and spikes.rate > 0.0:
            self.set_spikes(spikes)
            try:
                return self._quant_eval(images, calib, mode, d1, d2, spikes)
            finally:
                self.set_spikes(None)
        return self._quant_eval(images, calib, mode, d1, d2, None)

    def _quant_eval(self, images, calib, mode, d1, d2, spikes):
        import torch
        images = np.ascontiguousarray(images, np.float64)
        d = self.dims
        S, T, E, N = images.size // d.pix, d.tokens, d.embed, d.state
        lq = self.forward_host(images, calib, mode, d1=d1, d2=d2)
        lf = self.forward_host(images, None, L.MODE_FP, d1=d1, d2=d2)
        diff = lf - lq
        out = dict(logits_fp=lf, logits_q=lq, logits_mse=float(np.sum(diff * diff) / diff.size),
                   argmax_agree=int(np.sum(np.argmax(lf, axis=1) == np.argmax(lq, axis=1))), batch=S, layer_mse=[])
        scan, _ = calib.export()
        nd = len(self.orders)
        dev = torch.device("cuda", self.ctx.device)
        tdev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        for b in range(d.blocks):
            tr = self.trace(images, None, L.MODE_FP, b, d1=d1, d2=d2)
            u = tr.get("u", np.float64).reshape(S, T, E)
            for k, order in enumerate(self.orders):
                perm = _scan_perm(order, T, d.grid)
                # bypass re-scans with the unquantized model (quant.cpp:519-520: qmodel = model)
                pd = f"block{b}.dir{k}."
                wx = (np.concatenate([self.get_tensor(pd + n) for n in ("w_delta", "w_b", "w_c")]) if mode == L.MODE_FP
                      else self.qweight(pd + "xp", calib.spec.wbits))
                w = tdev(np.asarray(wx).reshape(E + 2 * N, E))
                proj = self.ctx.dgemm(tdev(u[:, perm, :].reshape(S * T, E)), w)  # k-ascending dots, as s6_scan
                o_tf = torch.empty(S * T * E, dtype=torch.float64, device=dev)
                tabs = [scan[(b * nd + k) * 3 + q] for q in range(3)]
                self.ctx.quant_scan(S=S, T=T, E=E, order=order, grid=d.grid, u=tdev(u), proj=proj,
                                    a=tdev(self.get_tensor(f"block{b}.dir{k}.a")),
                                    b_delta=tdev(self.get_tensor(f"block{b}.dir{k}.b_delta")), o=o_tf, mode=mode,
                                    n_refresh=calib.spec.n_refresh, act_bits=calib.spec.abits,
                                    outlier_bits=calib.spec.obits, theta=[t.theta for t in tabs],
                                    s_in=[tdev(t.s_in) for t in tabs], s_full=[tdev(t.s_full) for t in tabs],
                                    spikes=spikes, block=b, dir=k)
                e = tr.get(f"dir{k}.o", np.float64) - o_tf.cpu().numpy()
                out["layer_mse"].append((f"block{b}.dir{k}", float(np.sum(e * e) / e.size)))
        return out

    def trace(self, images: np.ndarray, calib: Calibration | None, mode: int, block: int, *, d1=True,
              d2=True) -> Trace:
        images = np.ascontiguousarray(images, np.float64)
        B = images.size // self.dims.pix
        h = C.c_void_p()
        L.check(self.lib.ouro_b200_trace_run(self.h, calib.h if calib else None, mode, int(d1), int(d2),
                                             _ptr(images), B, block, C.byref(h)))
        return Trace(self.lib, h)


# ---- OURO tensor files and pipeline stages (host-side entry points) -----------------

DTYPE_F64, DTYPE_I8, DTYPE_U4 = 0, 1, 2


def tensor_save(path, data: np.ndarray, dtype: int = DTYPE_F64, *, packed: bool = False, shape=None) -> None:
    """write_tensor_f64 / _i8 / _u4 (tensor_io.cpp) in the reference's OURO container.
    U4: int8 codes in [-8, 7], or (packed=True) the nibble-packed payload with `shape`
    the logical code shape (e.g. a K1 operand produced in the packed format)."""
    lib = L.load()
    arr = np.ascontiguousarray(data, np.float64 if dtype == DTYPE_F64 else (np.uint8 if packed else np.int8))
    shp = np.array(shape if shape is not None else arr.shape, dtype=np.uint64)
    L.check(lib.ouro_b200_tensor_save(str(path).encode(), dtype, _ptr(shp), shp.size, _ptr(arr), int(packed)))


def tensor_info(path):
    """(dtype, shape) of a tensor file."""
    lib = L.load()
    dt, rank = C.c_int(), C.c_size_t()
    shp = np.zeros(16, np.uint64)
    L.check(lib.ouro_b200_tensor_info(str(path).encode(), C.byref(dt), _ptr(shp), 16, C.byref(rank)))
    return dt.value, tuple(int(x) for x in shp[:rank.value])


def tensor_load(path, *, packed: bool = False) -> np.ndarray:
    """read_tensor_f64 / _i8 / _u4: f64 or int8 codes in the file's shape (packed=True: the raw u4 bytes)."""
    lib = L.load()
    dt, shape = tensor_info(path)
    n = int(np.prod(shape)) if shape else 1
    if dt == DTYPE_F64:
        out = np.empty(shape, np.float64)
    elif dt == DTYPE_U4 and packed:
        out = np.empty((n + 1) // 2, np.uint8)
    else:
        out = np.empty(shape, np.int8)
    L.check(lib.ouro_b200_tensor_load(str(path).encode(), dt, _ptr(out), out.nbytes, int(packed)))
    return out


@dataclass
class StageConfig:
    """The RunConfig settings the GPU stages read (config.hpp:17-47); scan orders
    row-forward, row-backward; d1 = d2 = False is the reference's own pass."""
    dims: Dims = field(default_factory=Dims)
    seed: int = 1
    weight_bits: int = 4
    act_bits: int = 8
    outlier_bits: int = 8
    n_refresh: int = 10
    outlier_quantile: float = 0.01
    mode: str = "dynamic"
    eval_batch: int = 4
    spike_rate: float = 0.0
    spike_gain: float = 100.0
    spike_channels: int = 1
    d1: bool = False
    d2: bool = False
    run_id: str | None = None
    device: int = 0

    def _c(self):
        d = self.dims
        self._mode_b = self.mode.encode()
        self._run_b = self.run_id.encode() if self.run_id is not None else None
        return L.StageConfig(d.image, d.channels, d.patch, d.embed, d.state, d.blocks, d.classes, d.conv_width,
                             self.seed, self.weight_bits, self.act_bits, self.outlier_bits, self.n_refresh,
                             self.outlier_quantile, self._mode_b, self.eval_batch, self.spike_rate, self.spike_gain,
                             self.spike_channels, int(self.d1), int(self.d2), self._run_b, self.device)


def quant_eval_stage(cfg: StageConfig, calib_dir, images_file, out_dir) -> None:
    """ouro_quant_eval (capi.cpp:174-186) on the GPU: writes out_dir/metrics.txt + manifest.txt."""
    lib = L.load()
    c = cfg._c()
    L.check(lib.ouro_b200_quant_eval(C.byref(c), str(calib_dir).encode(), str(images_file).encode(),
                                     str(out_dir).encode()))


def calib_stage(cfg: StageConfig, images_file, out_dir) -> None:
    """ouro_calib (capi.cpp:166-172) on the GPU: the calibration directory + manifest."""
    lib = L.load()
    c = cfg._c()
    L.check(lib.ouro_b200_calib_stage(C.byref(c), str(images_file).encode(), str(out_dir).encode()))
