// inst_f64_mp16.cu — the variant-2 launchers for T=double, MP=16 (inst_tma.cuh).
#include "inst_tma.cuh"

AD2_INST_TMA(double, 16)
