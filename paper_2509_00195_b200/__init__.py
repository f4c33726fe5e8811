"""B200-native hot path of FlashTTS's beam-search TTS step (arXiv 2509.00195).

libtts.so (C-ABI, include/tts.h) holds every kernel; ``tts`` is the ctypes
binding, ``runner`` drives a workload through it, ``metrics`` holds the byte
accounting used for the roofline.  This package never imports ``oracle``.
"""
from . import metrics  # noqa: F401
