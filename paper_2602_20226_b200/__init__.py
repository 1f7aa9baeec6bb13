"""B200-native zip-up (arXiv 2602.20226 hot path): libqtt.so C-ABI + thin binding.

Import submodules explicitly: ``gen`` (seeded inputs, numpy only) and ``qtt`` (the ctypes
binding of the CUDA library; needs torch and a built ``lib/libqtt.so``)."""
