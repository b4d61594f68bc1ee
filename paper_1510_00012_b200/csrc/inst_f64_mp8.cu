// inst_f64_mp8.cu — the variant-2 launchers for T=double, MP=8 (inst_tma.cuh).
#include "inst_tma.cuh"

AD2_INST_TMA(double, 8)
