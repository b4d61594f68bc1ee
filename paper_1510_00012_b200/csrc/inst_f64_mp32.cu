// inst_f64_mp32.cu — the variant-2 launchers for T=double, MP=32 (inst_tma.cuh).
#include "inst_tma.cuh"

AD2_INST_TMA(double, 32)
AD2_INST_COST_MEMBER(double)
