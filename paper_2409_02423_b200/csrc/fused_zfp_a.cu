// fused_zfp_a.cu -- NVLink engine kernels, zfp-rate 3..16 (see fused_launch.cuh).
#include "codec_zfp.cuh"
#include "fused_launch.cuh"

namespace hccx {

cudaError_t launch_fused_zfp_a(int rate, const FusedParams* p, int nv, cudaStream_t s) {
  switch (rate) {
    case 3: return launch_fused_codec<ZfpRateCodec<3>>(p, nv, s);
    case 4: return launch_fused_codec<ZfpRateCodec<4>>(p, nv, s);
    case 5: return launch_fused_codec<ZfpRateCodec<5>>(p, nv, s);
    case 6: return launch_fused_codec<ZfpRateCodec<6>>(p, nv, s);
    case 7: return launch_fused_codec<ZfpRateCodec<7>>(p, nv, s);
    case 8: return launch_fused_codec<ZfpRateCodec<8>>(p, nv, s);
    case 9: return launch_fused_codec<ZfpRateCodec<9>>(p, nv, s);
    case 10: return launch_fused_codec<ZfpRateCodec<10>>(p, nv, s);
    case 11: return launch_fused_codec<ZfpRateCodec<11>>(p, nv, s);
    case 12: return launch_fused_codec<ZfpRateCodec<12>>(p, nv, s);
    case 13: return launch_fused_codec<ZfpRateCodec<13>>(p, nv, s);
    case 14: return launch_fused_codec<ZfpRateCodec<14>>(p, nv, s);
    case 15: return launch_fused_codec<ZfpRateCodec<15>>(p, nv, s);
    case 16: return launch_fused_codec<ZfpRateCodec<16>>(p, nv, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hccx
