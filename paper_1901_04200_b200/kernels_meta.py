"""Compile-time constants of the CUDA kernels (csrc/kernels.h) that host-side
test code mirrors (the gloo sharding test's fixed-order reduction)."""
BLOCK = 128          # kBlock: threads per CTA, one path per thread
GROUP = 64           # kGroup: chunks per first-level reduction group (reduce.cu)
