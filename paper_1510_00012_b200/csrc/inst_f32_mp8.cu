// inst_f32_mp8.cu — the variant-2 launchers for T=float, MP=8 (inst_tma.cuh).
#include "inst_tma.cuh"

AD2_INST_TMA(float, 8)
