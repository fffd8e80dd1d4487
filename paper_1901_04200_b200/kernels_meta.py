"""Compile-time constants of the CUDA kernels (csrc/kernels.h), for host-side accounting."""
BLOCK = 128          # kBlock
SEG_STEPS = 16       # kSegSteps: steps per checkpoint segment
GROUP = 64           # kGroup: chunks per first-level reduction group
