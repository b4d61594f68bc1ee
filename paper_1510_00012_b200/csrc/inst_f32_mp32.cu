// inst_f32_mp32.cu — the variant-2 launchers for T=float, MP=32 (inst_tma.cuh).
#include "inst_tma.cuh"

AD2_INST_TMA(float, 32)
AD2_INST_COST_MEMBER(float)
