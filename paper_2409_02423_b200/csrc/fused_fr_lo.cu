// fused_fr_lo.cu -- NVLink engine kernels, fixed-rate 2..16 (see fused_launch.cuh).
#include "codec_fixed_rate.cuh"
#include "fused_launch.cuh"

namespace hccx {

cudaError_t launch_fused_fr_lo(int rate, const FusedParams* p, int nv, cudaStream_t s) {
  switch (rate) {
    case 2: return launch_fused_codec<FixedRateCodec<2>>(p, nv, s);
    case 3: return launch_fused_codec<FixedRateCodec<3>>(p, nv, s);
    case 4: return launch_fused_codec<FixedRateCodec<4>>(p, nv, s);
    case 5: return launch_fused_codec<FixedRateCodec<5>>(p, nv, s);
    case 6: return launch_fused_codec<FixedRateCodec<6>>(p, nv, s);
    case 7: return launch_fused_codec<FixedRateCodec<7>>(p, nv, s);
    case 8: return launch_fused_codec<FixedRateCodec<8>>(p, nv, s);
    case 9: return launch_fused_codec<FixedRateCodec<9>>(p, nv, s);
    case 10: return launch_fused_codec<FixedRateCodec<10>>(p, nv, s);
    case 11: return launch_fused_codec<FixedRateCodec<11>>(p, nv, s);
    case 12: return launch_fused_codec<FixedRateCodec<12>>(p, nv, s);
    case 13: return launch_fused_codec<FixedRateCodec<13>>(p, nv, s);
    case 14: return launch_fused_codec<FixedRateCodec<14>>(p, nv, s);
    case 15: return launch_fused_codec<FixedRateCodec<15>>(p, nv, s);
    case 16: return launch_fused_codec<FixedRateCodec<16>>(p, nv, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hccx
