"""CPU tests: byte accounting pins and the C-ABI library surface (no GPU calls)."""
import ctypes

import pytest

from paper_2509_00195_b200 import metrics


def test_kv_bytes_spec_example():
    # layers 2, kv_heads 2, head_dim 4, dtype 2, batch 1, seq 10 -> 640 B
    assert metrics.kv_bytes(2, 2, 4, 2, 1, 10) == 640
    assert metrics.kv_bytes(2, 2, 4, 2, 0, 10) == 0
    assert metrics.kv_bytes(2, 2, 4, 2, 2, 10) == 2 * metrics.kv_bytes(2, 2, 4, 2, 1, 10)


def test_t_roof_spec_examples():
    # SPEC S:331-334
    assert metrics.t_roof(1e12, 1e9, 1, 1) == 1.0
    assert metrics.t_roof(2e12, 1e9, 1, 1) == 2.0
    assert metrics.t_roof(1e12, 5e9, 1, 1) == 5.0


@pytest.fixture(scope="module")
def lib():
    from paper_2509_00195_b200 import build, tts
    build.build()
    return tts.load()


def test_library_exports_every_header_symbol(lib):
    from paper_2509_00195_b200 import tts
    names = tts.header_functions()
    assert "tts_prefix_attn_decode" in names and "tts_beam_select_fork" in names
    assert any(n.startswith("tts_block_table_") for n in names)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_query_buffer_bytes_host_only(lib):
    from paper_2509_00195_b200 import tts
    cfg = tts.TTSConfig(num_layers=2, num_q_heads=4, num_kv_heads=2, head_dim=64, page_size=16,
                        max_requests=1, max_beams=4, max_pages_per_beam=8, num_pages=100)
    s = tts.query_buffer_bytes(cfg)
    assert s["k_pool"] == 2 * 100 * 2 * 16 * 64 * 2
    assert s["block_tables"] == 1 * 4 * 8 * 4
    assert s["free_bitmap"] == 4 * 4
    bad = tts.TTSConfig(2, 5, 2, 64, 16, 1, 4, 8, 100)  # Hq % Hkv != 0
    with pytest.raises(tts.TTSError):
        tts.query_buffer_bytes(bad)
    assert lib.tts_status_str(3) == b"page pool exhausted"


def test_no_cpu_fallback(lib):
    import torch
    from paper_2509_00195_b200 import tts
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = tts.TTSConfig(1, 4, 2, 64, 16, 1, 4, 8, 100)
    with pytest.raises(RuntimeError):
        tts.Context(cfg)
