// cossin_b200.cu -- unity translation unit: one .so, one copy of the
// __constant__ tables shared by every kernel (no relocatable device code).
#include "k0_select.cu"
#include "fused64.cu"
#include "fused64d.cu"
#include "tiled.cu"
#include "distchain.cu"
#include "ddref.cu"
#include "residual.cu"
#include "abi.cu"
