// CUTLASS cross-check family table (tools/cutlass_xcheck/gen_family.py)
#include "wt_gemm.h"
#include "wt_gemm_table.inc"
