// inst_f32_mp16.cu — the variant-2 launchers for T=float, MP=16 (inst_tma.cuh).
#include "inst_tma.cuh"

AD2_INST_TMA(float, 16)
