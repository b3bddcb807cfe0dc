"""B200-native hot path of arXiv 2205.06327 (gradient decomposition + APPP).

The product is libptycho.so (include/ptycho.h); `paper_2205_06327_b200.ptycho` is its thin
ctypes binding.  Importing the binding requires the built extension (no fallback).
"""
