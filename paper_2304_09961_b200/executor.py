"""Python handle on libbs_exec.so (the B200 executor C-ABI, include/bs_exec.h).

Mirrors the reference's serving entry points: admit / step / retire / drop
at the points where batchsim's Simulator does arrive_at_server / start_step /
finish / drop (proj/include/batchsim/simulator.hpp:447-751), plus replay
(run_sim with every step executed), live serving and latency profiling.
There is no CPU fallback: without the CUDA library or a GPU these raise.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from ._native import BsError, FP, exec_lib, nets_check, nets_lib

_declared = False


class bs_member(C.Structure):
    _fields_ = [("id", C.c_int64), ("layer", C.c_int)]


class bs_rider(C.Structure):
    _fields_ = [("id", C.c_int64), ("dnn", C.c_int), ("join_layer", C.c_int),
                ("leave_layer", C.c_int), ("deposit_layer", C.c_int)]


class bs_step_result(C.Structure):
    _fields_ = [("layers_run", C.c_int), ("max_batch", C.c_int), ("kernels", C.c_int), ("done_event", C.c_void_p)]


def _lib():
    global _declared
    lib = exec_lib()
    if not _declared:
        H = C.c_void_p
        sig = {
            "bs_create": ([C.c_int, C.c_char_p, C.c_int, C.c_int, C.POINTER(H)], C.c_int),
            "bs_create_ex": ([C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(H)], C.c_int),
            "bs_step_ex": ([H, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(bs_member), C.c_int,
                            C.POINTER(bs_rider), C.c_int, C.c_void_p, C.POINTER(bs_step_result)], C.c_int),
            "bs_destroy": ([H], C.c_int),
            "bs_suite_json": ([H, C.POINTER(C.c_void_p)], C.c_int),
            "bs_read_weights": ([H, FP, C.c_size_t], C.c_int),
            "bs_admit": ([H, C.c_int64, C.c_int, C.c_int, FP], C.c_int),
            "bs_admit_device": ([H, C.c_int64, C.c_int, C.c_void_p], C.c_int),
            "bs_plan": ([H, C.c_int], C.c_int),
            "bs_step": ([H, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(bs_member), C.c_int,
                         C.POINTER(bs_rider), C.c_int], C.c_int),
            "bs_step_done": ([H, C.POINTER(C.c_int64), C.c_int], C.c_int),
            "bs_retire": ([H, C.c_int64, FP, C.c_int, C.c_int], C.c_int),
            "bs_drop": ([H, C.c_int64], C.c_int),
            "bs_read_blob": ([H, C.c_int64, FP, C.c_size_t], C.c_int),
            "bs_sync": ([H], C.c_int),
            "bs_profile_layer": ([H, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)], C.c_int),
            "bs_profile_span": ([H, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)], C.c_int),
            "bs_profile_table": ([H, C.c_char_p, C.POINTER(C.c_void_p)], C.c_int),
            "bs_replay": ([H, C.c_char_p, C.POINTER(C.c_void_p)], C.c_int),
            "bs_serve": ([H, C.c_char_p, C.POINTER(C.c_void_p)], C.c_int),
            "bs_free": ([C.c_void_p], None),
            "bs_set_precision": ([H, C.c_char_p], C.c_int),
            "bs_stats": ([H, C.c_int, C.c_int], C.c_int),
            "bs_stats_summary": ([H, C.c_double, C.c_double, C.POINTER(C.c_void_p)], C.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        _declared = True
    return lib


def _check(rc):
    if rc != 0:
        msg = _lib().bs_last_error()
        text = msg.decode() if msg else ""
        if rc == -1:
            raise ValueError(text)
        if rc in (-4, -5):
            raise RuntimeError(f"logic_error: {text}")
        raise BsError(f"status {rc}: {text}")


def _take_string(ptr: C.c_void_p) -> str:
    try:
        return C.string_at(ptr).decode()
    finally:
        _lib().bs_free(ptr)


def describe_suite(suite: str) -> dict:
    """Network description of a suite, built on the host (libbs_nets.so, no GPU needed)."""
    lib = nets_lib()
    out = C.c_void_p()
    nets_check(lib.bs_describe_suite(suite.encode(), C.byref(out)))
    try:
        return json.loads(C.string_at(out).decode())
    finally:
        lib.bs_nets_free(out)


def suite_weights(suite: str, desc: dict | None = None) -> np.ndarray:
    """The suite's calibrated weight pool, built on the host (libbs_nets.so)."""
    desc = desc or describe_suite(suite)
    w = np.empty(desc["weights"], np.float32)
    nets_check(nets_lib().bs_suite_weights_host(suite.encode(), w.ctypes.data_as(FP), w.size))
    return w


def make_image(seed: int, index: int, H: int, W: int, C_: int, real_c: int = 3) -> np.ndarray:
    out = np.empty((H, W, C_), np.float32)
    nets_check(nets_lib().bs_make_image(seed, index, H, W, C_, real_c, out.ctypes.data_as(FP)))
    return out


class Executor:
    def __init__(self, suite: str, device: int = 0, max_batch: int = 90, max_requests: int = 1024,
                 window_cap: int | None = None, dtype: str | None = None):
        h = C.c_void_p()
        if window_cap is None and dtype is None:
            _check(_lib().bs_create(device, suite.encode(), max_batch, max_requests, C.byref(h)))
        else:  # the SURVEY.md §8(b) form
            _check(_lib().bs_create_ex(device, suite.encode(), max_batch, max_requests, window_cap or 0,
                                       dtype.encode() if dtype else None, C.byref(h)))
        self._h = h
        self.suite_name = suite
        self.max_batch = max_batch
        self._desc = None

    def set_precision(self, mode: str):
        """"tf32x2" (default, fp32 parity) or "tf32"."""
        _check(_lib().bs_set_precision(self._h, mode.encode()))

    def close(self):
        if self._h:
            _check(_lib().bs_destroy(self._h))
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- model
    @property
    def desc(self) -> dict:
        if self._desc is None:
            out = C.c_void_p()
            _check(_lib().bs_suite_json(self._h, C.byref(out)))
            self._desc = json.loads(_take_string(out))
        return self._desc

    def weights(self) -> np.ndarray:
        w = np.empty(self.desc["weights"], np.float32)
        _check(_lib().bs_read_weights(self._h, w.ctypes.data_as(FP), w.size))
        return w

    def dnn_index(self, name: str) -> int:
        return [n["name"] for n in self.desc["nets"]].index(name)

    # ------------------------------------------------------------- requests
    def admit(self, rid: int, dnn: int, image: np.ndarray, entry_layer: int = 1):
        image = np.ascontiguousarray(image, np.float32)
        _check(_lib().bs_admit(self._h, rid, dnn, entry_layer, image.ctypes.data_as(FP)))

    def admit_device(self, rid: int, dnn: int, image_ptr: int):
        """Admit with the NHWC fp32 input already in device memory (e.g. a
        torch CUDA tensor's data_ptr()): read in place by the first layer, so
        it must outlive that layer."""
        _check(_lib().bs_admit_device(self._h, rid, dnn, C.c_void_p(image_ptr)))

    def admit_rgb_many(self, rids, dnn: int, images):
        """Admit k arrivals of one DNN shipped as packed 8-bit RGB [H][W][3]
        uint8 arrays (bs_admit_rgb_many: one packed H2D copy and one
        expansion launch for the batch)."""
        import numpy as np
        arrs = [np.ascontiguousarray(im, dtype=np.uint8) for im in images]
        k = len(arrs)
        ids = (C.c_int64 * k)(*rids)
        ptrs = (C.c_void_p * k)(*[a.ctypes.data for a in arrs])
        _check(_lib().bs_admit_rgb_many(self._h, ids, dnn, ptrs, k))

    def plan(self, plan_no: int):
        _check(_lib().bs_plan(self._h, plan_no))

    def step(self, plan_no: int, segment: int, dnn: int, layer_from: int, layer_to: int,
             members: list[tuple[int, int]], riders: list[tuple] = ()):
        m = (bs_member * max(1, len(members)))(*[bs_member(i, l) for i, l in members])
        r = (bs_rider * max(1, len(riders)))(*[bs_rider(*x) for x in riders])
        _check(_lib().bs_step(self._h, plan_no, segment, dnn, layer_from, layer_to, m, len(members), r,
                              len(riders)))

    def step_ex(self, plan_no: int, segment: int, dnn: int, layer_from: int, layer_to: int,
                members: list[tuple[int, int]], riders: list[tuple] = (), stream: int | None = None) -> dict:
        """bs_step_ex: ordered after / awaited by `stream` (a cudaStream_t as an
        int, or None); returns the step result (done_event = cudaEvent_t)."""
        m = (bs_member * max(1, len(members)))(*[bs_member(i, l) for i, l in members])
        r = (bs_rider * max(1, len(riders)))(*[bs_rider(*x) for x in riders])
        res = bs_step_result()
        _check(_lib().bs_step_ex(self._h, plan_no, segment, dnn, layer_from, layer_to, m, len(members), r,
                                 len(riders), C.c_void_p(stream) if stream else None, C.byref(res)))
        return {"layers_run": res.layers_run, "max_batch": res.max_batch, "kernels": res.kernels,
                "done_event": res.done_event}

    def step_done(self, deposited: list[int]):
        arr = (C.c_int64 * max(1, len(deposited)))(*deposited)
        _check(_lib().bs_step_done(self._h, arr, len(deposited)))

    def retire(self, rid: int, n: int, logits: bool = False) -> np.ndarray:
        out = np.empty(n, np.float32)
        _check(_lib().bs_retire(self._h, rid, out.ctypes.data_as(FP), n, int(logits)))
        return out

    def drop(self, rid: int):
        _check(_lib().bs_drop(self._h, rid))

    def read_blob(self, rid: int) -> np.ndarray:
        out = np.empty(self.desc["slot_floats"], np.float32)
        _check(_lib().bs_read_blob(self._h, rid, out.ctypes.data_as(FP), out.size))
        return out

    def sync(self):
        _check(_lib().bs_sync(self._h))

    # ---------------------------------------------------------- measurement
    def profile_layer(self, dnn: int, layer: int, batch: int, reps: int = 10, flush_l2: bool = False) -> float:
        ms = C.c_double()
        _check(_lib().bs_profile_layer(self._h, dnn, layer, batch, reps, int(flush_l2), C.byref(ms)))
        return ms.value

    def profile_table(self, batches=(1, 2, 4, 8, 16, 32, 64, 90), reps: int = 10, flush_l2: bool = False,
                      tune_tiles: bool = False, timing: str = "step") -> dict:
        """Measured h_k(b) table in the reference schema. tune_tiles: first
        autotune every conv's launch choices per batch -- K split, tile width,
        grouped vs separate conv pairs -- (kept for later launches; timings
        returned under "tile_tune"). timing: "step" (default) = each layer as
        a one-layer serving step inside back-to-back passes run as such steps
        (device-stamped), "pass" = each layer inside back-to-back network
        passes with events between layers, scaled to the whole-pass time,
        "layer" = each layer alone, synchronised. flush_l2: cold-L2 layer
        timings (per-layer mode)."""
        out = C.c_void_p()
        opts = json.dumps({"batches": list(batches), "reps": reps, "flush_l2": bool(flush_l2),
                           "tune_tiles": bool(tune_tiles), "timing": timing})
        _check(_lib().bs_profile_table(self._h, opts.encode(), C.byref(out)))
        return json.loads(_take_string(out))

    def profile_span(self, dnn: int, lo: int, hi: int, batch: int, reps: int = 20) -> tuple[float, float, float]:
        """ms per pass of layers [lo, hi] at `batch`: (synchronised, back to back, CUDA graph)."""
        out = (C.c_double * 3)()
        _check(_lib().bs_profile_span(self._h, dnn, lo, hi, batch, reps, out))
        return out[0], out[1], out[2]

    def stats(self, enable: bool, every: int = 1):
        _check(_lib().bs_stats(self._h, int(enable), every))

    def stats_summary(self, hbm_gbs: float, tensor_tflops: float) -> dict:
        out = C.c_void_p()
        _check(_lib().bs_stats_summary(self._h, hbm_gbs, tensor_tflops, C.byref(out)))
        return json.loads(_take_string(out))

    # -------------------------------------------------------------- serving
    def replay(self, job: dict) -> list[dict]:
        out = C.c_void_p()
        _check(_lib().bs_replay(self._h, json.dumps(dict(job, job="sim")).encode(), C.byref(out)))
        return [json.loads(l) for l in _take_string(out).splitlines()]

    def serve(self, job: dict) -> dict:
        out = C.c_void_p()
        _check(_lib().bs_serve(self._h, json.dumps(dict(job, job="sim")).encode(), C.byref(out)))
        return json.loads(_take_string(out))
