"""PrefillShare hot path, B200-native (sm_100a).

One frozen prefill module writes a paged prompt KV cache once; N decode
modules reuse it. Host side: Python mirrors of the reference API
(kvstore.BlockPool, router.Router, model modules); compute: libpsk.so
(hand-written CUDA for sm_100a behind the C ABI in include/psk.h).
"""

__version__ = "0.1.0"
