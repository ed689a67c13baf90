// tma_host.h -- host side of TMA tensor maps: cuTensorMapEncodeTiled through the
// runtime's driver entry point (the library links cudart statically, not libcuda).
#pragma once
#include <cuda.h>

namespace ephdc {

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// nullptr if the driver does not provide it
EncodeTiledFn encode_tiled_fn();

}  // namespace ephdc
