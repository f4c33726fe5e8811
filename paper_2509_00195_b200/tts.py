"""Thin ctypes binding of libtts (include/tts.h).  Argument marshalling only:
every step of the hot path runs in the CUDA kernels behind the C-ABI.  The
functions carry the C names; ``Context`` owns the caller-side device buffers.

There is no fallback: if libtts.so is missing or no CUDA device is present,
constructing a Context raises.
"""
from __future__ import annotations

import ctypes
import os
import re
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TTS_LIB_PATH") or os.path.join(HERE, "libtts.so")  # override: variant builds (tools/)
HEADER = os.path.join(os.path.dirname(HERE), "include", "tts.h")


SELECT_TOPK, SELECT_DIVERSE, SELECT_DYNAMIC = 0, 1, 2  # include/tts.h


class TTSError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        super().__init__(f"{what}: libtts status {code} ({status_str(code)})")


class tts_config_t(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("page_size", ctypes.c_int32), ("max_requests", ctypes.c_int32),
                ("max_beams", ctypes.c_int32), ("max_pages_per_beam", ctypes.c_int32),
                ("num_pages", ctypes.c_int64)]


class tts_buffers_t(ctypes.Structure):
    _fields_ = [("k_pool", ctypes.c_void_p), ("v_pool", ctypes.c_void_p),
                ("block_tables", ctypes.c_void_p), ("seq_lens", ctypes.c_void_p),
                ("refcounts", ctypes.c_void_p), ("free_bitmap", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t)]


class tts_buffer_sizes_t(ctypes.Structure):
    _fields_ = [(n, ctypes.c_size_t) for n in ("k_pool", "v_pool", "block_tables", "seq_lens",
                                               "refcounts", "free_bitmap", "status", "workspace")]


_lib = None
_P = ctypes.c_void_p
_I = ctypes.c_int32

# host transport callbacks (include/tts.h tts_host_transport_t)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, _P, _P, _P, ctypes.c_size_t)
SENDRECV_FN = ctypes.CFUNCTYPE(ctypes.c_int, _P, _I, ctypes.POINTER(_I), ctypes.POINTER(_P),
                               ctypes.POINTER(ctypes.c_size_t), _I, ctypes.POINTER(_I), ctypes.POINTER(_P),
                               ctypes.POINTER(ctypes.c_size_t))


class tts_host_transport_t(ctypes.Structure):
    _fields_ = [("user", _P), ("allgather", ALLGATHER_FN), ("sendrecv", SENDRECV_FN)]


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -m paper_2509_00195_b200.build` "
                               "or __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        sig = {
            "tts_query_buffer_bytes": [ctypes.POINTER(tts_config_t), ctypes.POINTER(tts_buffer_sizes_t)],
            "tts_create": [ctypes.POINTER(tts_config_t), ctypes.POINTER(tts_buffers_t), ctypes.c_int, ctypes.POINTER(_P)],
            "tts_destroy": [_P],
            "tts_device_status": [_P, _P, ctypes.POINTER(ctypes.c_int)],
            "tts_block_table_init_request": [_P, _I, _I, _I, _P, _P, _P],
            "tts_block_table_append": [_P, _I, _P, _P, _P, _P, _P],
            "tts_prefix_attn_decode": [_P, _I, _I, _I, _P, _P, _P, ctypes.c_float, _P, _P],
            "tts_beam_select_fork": [_P, _I, _P, _P, _I, _P, _P],
            "tts_beam_select_fork_policy": [_P, _I, _P, _P, _I, _I, _P, _P],
            "tts_block_table_release_request": [_P, _I, _P],
            "tts_block_table_snapshot": [_P, _I, _P, _P, _P, _P, _P, _P],
            "tts_block_table_stats": [_P, _I, _P, _P, _P, _P],
            "tts_seq_lens_host": [_P, _I, _P],
            "tts_decode_step": [_P, _I, _P, _P, _P, _P, _P, ctypes.c_float, _P, _P],
            "tts_profile_begin": [_P],
            "tts_profile_end": [_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)],
            "tts_beam_select_global": [_P, _I, _P, _I, _P, _P],
            "tts_beam_fork_map": [_P, _I, _I, _P, _P],
            "tts_lineage_bytes": [_P, _I, ctypes.POINTER(ctypes.c_size_t)],
            "tts_lineage_export": [_P, _I, _I, _P, _P],
            "tts_lineage_import": [_P, _I, _I, _I, _P, _P],
            "tts_comm_unique_id": [_P],
            "tts_comm_init": [_P, _P, _I, _I, _P, ctypes.c_size_t],
            "tts_comm_init_host": [_P, _I, _I, ctypes.POINTER(tts_host_transport_t), ctypes.c_size_t],
            "tts_comm_destroy": [_P],
            "tts_span_init": [_P, _I, _I, _P, _I],
            "tts_span_stats": [_P, _I, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)],
            "tts_span_gids": [_P, _I, _P],
            "tts_beam_select_fork_global": [_P, _I, _P, _I, _P, _P, _P],
            "tts_span_placement": [_I, _P, _P, _I, _P, _P],
            "tts_spec_select": [_I, _P, _P, _P, _I, _I, _P],
            "tts_spec_branch": [_P, _I, _I, _P, _P],
            "tts_spec_plan": [_I, _I, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P],
            "tts_beam_fork_map_trunc": [_P, _I, _I, _P, _P, _P],
            "tts_dpas_plan": [_P, _I, ctypes.c_int64, _P, _P, _P, _P, _P, _P, _P],
        }
        for name, args in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        lib.tts_status_str.argtypes = [ctypes.c_int]
        lib.tts_status_str.restype = ctypes.c_char_p
        lib.tts_launch_count.argtypes = [_P]
        lib.tts_launch_count.restype = ctypes.c_int64
        lib.tts_attention_kernel.argtypes = [_P]
        lib.tts_attention_kernel.restype = ctypes.c_char_p
        lib.tts_stream_read_gbs.argtypes = [_P, ctypes.c_size_t, _I, ctypes.POINTER(ctypes.c_double), _P]
        lib.tts_stream_read_gbs.restype = ctypes.c_int
        _lib = lib
    return _lib


def header_functions() -> list:
    """Function names declared in include/tts.h (for the export test)."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tts_[a-z0-9_]+)\s*\(", src)))


def comm_unique_id() -> bytes:
    """tts_comm_unique_id: a fresh 128-byte NCCL unique id (rank 0 broadcasts it)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().tts_comm_unique_id(ctypes.cast(buf, _P)), "tts_comm_unique_id")
    return buf.raw


def span_placement(parent_gid: Sequence[int], old_rank: Sequence[int], caps: Sequence[int]) -> list:
    """tts_span_placement (host only): child gid -> rank."""
    n = len(parent_gid)
    out = (_I * n)()
    _check(load().tts_span_placement(n, _i32_host(parent_gid), _i32_host(old_rank), len(caps), _i32_host(caps),
                                     out), "tts_span_placement")
    return list(out)


def spec_select(beams: Sequence[int], last_scores: Sequence[float], have: Sequence[int], free_slots: int,
                B: int) -> list:
    """tts_spec_select (host only): new speculative branches per candidate."""
    n = len(beams)
    sc = (ctypes.c_float * max(1, n))(*[float(x) for x in last_scores])
    out = (_I * max(1, n))()
    _check(load().tts_spec_select(n, _i32_host(beams), sc, _i32_host(have), int(free_slots), int(B), out),
           "tts_spec_select")
    return list(out)[:n]


def spec_plan(parent: Sequence[int], M: int, branches: Sequence, lens: Sequence[int], frac: Sequence[float],
              next_len: Optional[Sequence[int]] = None):
    """tts_spec_plan (host only): (parent_rows, new_lens, head) of DuplicateThenTruncate."""
    N = len(parent)
    nb = len(branches)
    fr = (ctypes.c_double * N)(*[float(x) for x in frac])
    pr, nl, hd = (_I * N)(), (_I * N)(), (_I * N)()
    _check(load().tts_spec_plan(N, int(M), _i32_host(parent), nb, _i32_host([b[0] for b in branches] or [0]),
                                _i32_host([b[1] for b in branches] or [0]), _i32_host(lens), fr,
                                None if next_len is None else _i32_host(next_len), pr, nl, hd), "tts_spec_plan")
    return list(pr), list(nl), list(hd)


def stream_read_gbs(buf: torch.Tensor, iters: int = 10) -> float:
    """tts_stream_read_gbs: HBM read bandwidth over the device tensor buf (syncs)."""
    g = ctypes.c_double()
    st = ctypes.c_void_p(torch.cuda.current_stream(buf.device).cuda_stream)
    _check(load().tts_stream_read_gbs(ctypes.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size(),
                                      int(iters), ctypes.byref(g), st), "tts_stream_read_gbs")
    return g.value


def status_str(code: int) -> str:
    try:
        return load().tts_status_str(code).decode()
    except Exception:
        return "?"


def _check(code: int, what: str) -> None:
    if code != 0:
        raise TTSError(code, what)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _i32_host(xs: Sequence[int]):
    a = (ctypes.c_int32 * len(xs))(*[int(x) for x in xs])
    return a


def _u8_host(active: Optional[np.ndarray]):
    if active is None:
        return None, None
    a = np.ascontiguousarray(active, dtype=np.uint8)
    return a, a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class TTSConfig:
    num_layers: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    page_size: int
    max_requests: int
    max_beams: int
    max_pages_per_beam: int
    num_pages: int

    def c(self) -> tts_config_t:
        return tts_config_t(self.num_layers, self.num_q_heads, self.num_kv_heads, self.head_dim,
                            self.page_size, self.max_requests, self.max_beams,
                            self.max_pages_per_beam, self.num_pages)


def query_buffer_bytes(cfg: TTSConfig) -> dict:
    s = tts_buffer_sizes_t()
    c = cfg.c()
    _check(load().tts_query_buffer_bytes(ctypes.byref(c), ctypes.byref(s)), "tts_query_buffer_bytes")
    return {n: getattr(s, n) for n, _ in tts_buffer_sizes_t._fields_}


class Context:
    """Owns the caller-side device buffers (torch) and the libtts context."""

    def __init__(self, cfg: TTSConfig, device: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("libtts needs a CUDA device (no CPU fallback)")
        lib = load()
        self.lib = lib
        self.cfg = cfg
        self.device = torch.device("cuda", device)
        sz = query_buffer_bytes(cfg)
        dev = self.device

        def buf(n, dtype=torch.uint8):
            return torch.empty(max(int(n), 16) // torch.tensor([], dtype=dtype).element_size(),
                               dtype=dtype, device=dev)

        self.k_pool = buf(sz["k_pool"], torch.bfloat16)
        self.v_pool = buf(sz["v_pool"], torch.float16)  # V is held in fp16 (include/tts.h)
        self.block_tables = buf(sz["block_tables"], torch.int32)
        self.seq_lens = buf(sz["seq_lens"], torch.int32)
        self.refcounts = buf(sz["refcounts"], torch.int32)
        self.free_bitmap = buf(sz["free_bitmap"], torch.int32)
        self.status = buf(sz["status"], torch.int32)
        self.workspace = buf(sz["workspace"], torch.uint8)
        b = tts_buffers_t(self.k_pool.data_ptr(), self.v_pool.data_ptr(), self.block_tables.data_ptr(),
                          self.seq_lens.data_ptr(), self.refcounts.data_ptr(),
                          self.free_bitmap.data_ptr(), self.status.data_ptr(),
                          self.workspace.data_ptr(), self.workspace.numel())
        h = ctypes.c_void_p()
        c = cfg.c()
        torch.cuda.synchronize(dev)
        _check(lib.tts_create(ctypes.byref(c), ctypes.byref(b), device, ctypes.byref(h)), "tts_create")
        self.h = h

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.tts_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def launch_count(self) -> int:
        return int(self.lib.tts_launch_count(self.h))

    def attention_kernel(self) -> str:
        return self.lib.tts_attention_kernel(self.h).decode()

    # -- C entry points (same names) ------------------------------------------
    def tts_block_table_init_request(self, req, n_beams, prompt_len, k_prompt, v_prompt):
        _check(self.lib.tts_block_table_init_request(self.h, req, n_beams, prompt_len, _ptr(k_prompt),
                                                     _ptr(v_prompt), self.stream),
               "tts_block_table_init_request")

    def tts_block_table_append(self, req_ids, active, k_new, v_new):
        _a, ap = _u8_host(active)
        _check(self.lib.tts_block_table_append(self.h, len(req_ids), _i32_host(req_ids), ap,
                                               _ptr(k_new), _ptr(v_new), self.stream),
               "tts_block_table_append")

    def tts_prefix_attn_decode(self, layer_begin, layer_end, req_ids, active, q, scale, out):
        _a, ap = _u8_host(active)
        _check(self.lib.tts_prefix_attn_decode(self.h, layer_begin, layer_end, len(req_ids),
                                               _i32_host(req_ids), ap, _ptr(q), float(scale),
                                               _ptr(out), self.stream),
               "tts_prefix_attn_decode")

    def tts_decode_step(self, req_ids, active, k_new, v_new, q, scale, out):
        _a, ap = _u8_host(active)
        _check(self.lib.tts_decode_step(self.h, len(req_ids), _i32_host(req_ids), ap, _ptr(k_new),
                                        _ptr(v_new), _ptr(q), float(scale), _ptr(out), self.stream),
               "tts_decode_step")

    def tts_profile_begin(self):
        _check(self.lib.tts_profile_begin(self.h), "tts_profile_begin")

    def tts_profile_end(self):
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        _check(self.lib.tts_profile_end(self.h, ctypes.byref(ms), ctypes.byref(n)), "tts_profile_end")
        return ms.value, n.value

    def tts_beam_select_fork(self, req_ids, scores, width_m, parent_out=None):
        _check(self.lib.tts_beam_select_fork(self.h, len(req_ids), _i32_host(req_ids), _ptr(scores),
                                             int(width_m), _ptr(parent_out), self.stream),
               "tts_beam_select_fork")

    def tts_beam_select_fork_policy(self, req_ids, scores, policy, param, parent_out=None):
        _check(self.lib.tts_beam_select_fork_policy(self.h, len(req_ids), _i32_host(req_ids), _ptr(scores),
                                                    int(policy), int(param), _ptr(parent_out), self.stream),
               "tts_beam_select_fork_policy")

    def tts_beam_select_global(self, scores_all, width_m, parent_gid_out):
        _check(self.lib.tts_beam_select_global(self.h, scores_all.numel(), _ptr(scores_all), int(width_m),
                                               _ptr(parent_gid_out), self.stream), "tts_beam_select_global")

    def tts_beam_fork_map(self, req, parent_local):
        arr = _i32_host(parent_local)
        _check(self.lib.tts_beam_fork_map(self.h, req, len(parent_local), arr, self.stream), "tts_beam_fork_map")

    def tts_dpas_plan(self, req, budget_pages, active=None):
        """-> (order, trie_of [n_beams], n_tries, cost, shared)."""
        n = self.n_beams(req)
        order = (_I * n)()
        trie = (_I * n)(*([-1] * n))
        nt = ctypes.c_int32()
        cost, shared = ctypes.c_int64(), ctypes.c_int64()
        _a, ap = _u8_host(active)
        _check(self.lib.tts_dpas_plan(self.h, req, int(budget_pages), ap, order, trie, ctypes.byref(nt),
                                      ctypes.byref(cost), ctypes.byref(shared), self.stream), "tts_dpas_plan")
        k = n if active is None else int(np.asarray(active).astype(bool).sum())
        return list(order)[:k], list(trie), nt.value, cost.value, shared.value

    def tts_spec_branch(self, req, src_rows):
        _check(self.lib.tts_spec_branch(self.h, req, len(src_rows), _i32_host(src_rows), self.stream),
               "tts_spec_branch")

    def tts_beam_fork_map_trunc(self, req, parent_rows, new_lens):
        _check(self.lib.tts_beam_fork_map_trunc(self.h, req, len(parent_rows), _i32_host(parent_rows),
                                                _i32_host(new_lens), self.stream), "tts_beam_fork_map_trunc")

    def tts_lineage_bytes(self, length) -> int:
        n = ctypes.c_size_t()
        _check(self.lib.tts_lineage_bytes(self.h, int(length), ctypes.byref(n)), "tts_lineage_bytes")
        return n.value

    def tts_lineage_export(self, req, beam, buf):
        _check(self.lib.tts_lineage_export(self.h, req, beam, _ptr(buf), self.stream), "tts_lineage_export")

    def tts_lineage_import(self, req, beam, length, buf):
        _check(self.lib.tts_lineage_import(self.h, req, beam, int(length), _ptr(buf), self.stream),
               "tts_lineage_import")

    def lineage_buffer(self, length) -> torch.Tensor:
        return torch.empty(max(16, self.tts_lineage_bytes(length)), dtype=torch.uint8, device=self.device)

    def sync(self):
        torch.cuda.current_stream(self.device).synchronize()

    # -- a8: libtts-owned communicator ---------------------------------------------
    def tts_comm_init(self, unique_id: bytes, nranks: int, rank: int, stage: torch.Tensor):
        idb = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(self.lib.tts_comm_init(self.h, ctypes.cast(idb, _P), nranks, rank, _ptr(stage),
                                      stage.numel() * stage.element_size()), "tts_comm_init")
        self._stage = stage

    def tts_comm_init_host(self, nranks: int, rank: int, transport, stage_bytes: int = 64 << 20):
        """transport: object with allgather(send: bytes, nbytes) -> bytes (all ranks, rank order) and
        sendrecv(sends: [(dst, bytes)], recvs: [(src, nbytes)]) -> [bytes]."""
        def ag(user, send_h, recv_h, nbytes):
            try:
                data = transport.allgather(ctypes.string_at(send_h, nbytes), nbytes)
                ctypes.memmove(recv_h, data, len(data))
                return 0
            except Exception:  # noqa: BLE001 -- reported to libtts as a transport failure
                import traceback
                traceback.print_exc()
                return 1

        def sr(user, n_send, dst, send_h, send_b, n_recv, src, recv_h, recv_b):
            try:
                sends = [(dst[i], ctypes.string_at(send_h[i], send_b[i])) for i in range(n_send)]
                recvs = [(src[i], recv_b[i]) for i in range(n_recv)]
                got = transport.sendrecv(sends, recvs)
                for i in range(n_recv):
                    ctypes.memmove(recv_h[i], got[i], recv_b[i])
                return 0
            except Exception:  # noqa: BLE001
                import traceback
                traceback.print_exc()
                return 1

        self._transport = (transport, ALLGATHER_FN(ag), SENDRECV_FN(sr))
        t = tts_host_transport_t(None, self._transport[1], self._transport[2])
        self._transport_struct = t
        _check(self.lib.tts_comm_init_host(self.h, nranks, rank, ctypes.byref(t), int(stage_bytes)),
               "tts_comm_init_host")

    def tts_comm_destroy(self):
        _check(self.lib.tts_comm_destroy(self.h), "tts_comm_destroy")

    def tts_span_init(self, req: int, n_global: int, caps: Sequence[int], dedup: bool = False):
        _check(self.lib.tts_span_init(self.h, req, n_global, _i32_host(caps), int(bool(dedup))), "tts_span_init")

    def tts_span_stats(self, req: int):
        """-> (bytes this rank sent for migrations, bytes deduplication saved it)."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(self.lib.tts_span_stats(self.h, req, ctypes.byref(a), ctypes.byref(b)), "tts_span_stats")
        return a.value, b.value

    def tts_span_gids(self, req: int) -> list:
        n = int(self.n_beams(req))
        out = (_I * max(1, n))()
        _check(self.lib.tts_span_gids(self.h, req, out), "tts_span_gids")
        return list(out)[:n]

    def n_beams(self, req: int) -> int:
        """Beam count of an installed request (through the snapshot call; syncs)."""
        n = ctypes.c_int32()
        tables = np.empty((self.cfg.max_beams, self.cfg.max_pages_per_beam), dtype=np.int32)
        lens = np.empty(self.cfg.max_beams, dtype=np.int32)
        _check(self.lib.tts_block_table_snapshot(self.h, req, ctypes.byref(n), tables.ctypes.data_as(_P),
                                                 lens.ctypes.data_as(_P), None, None, self.stream),
               "tts_block_table_snapshot")
        return n.value

    def tts_beam_select_fork_global(self, req: int, local_scores: torch.Tensor, width_m: int,
                                    parent_gid_out: Optional[torch.Tensor] = None,
                                    child_rank_out: Optional[torch.Tensor] = None):
        _check(self.lib.tts_beam_select_fork_global(self.h, req, _ptr(local_scores), int(width_m),
                                                    _ptr(parent_gid_out), _ptr(child_rank_out), self.stream),
               "tts_beam_select_fork_global")

    def tts_block_table_release_request(self, req):
        _check(self.lib.tts_block_table_release_request(self.h, req, self.stream),
               "tts_block_table_release_request")

    def tts_block_table_snapshot(self, req, with_pool_state=True):
        c = self.cfg
        n = ctypes.c_int32()
        tables = np.empty((c.max_beams, c.max_pages_per_beam), dtype=np.int32)
        lens = np.empty(c.max_beams, dtype=np.int32)
        ref = np.empty(c.num_pages, dtype=np.int32) if with_pool_state else None
        bm = np.empty((c.num_pages + 31) // 32, dtype=np.uint32) if with_pool_state else None
        _check(self.lib.tts_block_table_snapshot(
            self.h, req, ctypes.byref(n), tables.ctypes.data_as(_P), lens.ctypes.data_as(_P),
            None if ref is None else ref.ctypes.data_as(_P), None if bm is None else bm.ctypes.data_as(_P),
            self.stream), "tts_block_table_snapshot")
        N = n.value
        out = {"n_beams": N, "tables": tables[:N], "lens": lens[:N]}
        if with_pool_state:
            out["ref"] = ref
            bits = np.unpackbits(bm.view(np.uint8), bitorder="little")[: c.num_pages]
            out["free"] = np.nonzero(bits)[0]
        return out

    def tts_block_table_stats(self, req_ids, active, accum):
        _a, ap = _u8_host(active)
        _check(self.lib.tts_block_table_stats(self.h, len(req_ids), _i32_host(req_ids), ap, _ptr(accum),
                                              self.stream), "tts_block_table_stats")

    def tts_device_status(self) -> int:
        v = ctypes.c_int()
        _check(self.lib.tts_device_status(self.h, self.stream, ctypes.byref(v)), "tts_device_status")
        return v.value

    def tts_seq_lens_host(self, req) -> np.ndarray:
        out = np.empty(self.cfg.max_beams, dtype=np.int32)
        _check(self.lib.tts_seq_lens_host(self.h, req, out.ctypes.data_as(_P)), "tts_seq_lens_host")
        return out
