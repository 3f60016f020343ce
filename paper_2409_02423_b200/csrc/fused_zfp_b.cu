// fused_zfp_b.cu -- NVLink engine kernels, zfp-rate 17..32 (see fused_launch.cuh).
#include "codec_zfp.cuh"
#include "fused_launch.cuh"

namespace hccx {

cudaError_t launch_fused_zfp_b(int rate, const FusedParams* p, int nv, cudaStream_t s) {
  switch (rate) {
    case 17: return launch_fused_codec<ZfpRateCodec<17>>(p, nv, s);
    case 18: return launch_fused_codec<ZfpRateCodec<18>>(p, nv, s);
    case 19: return launch_fused_codec<ZfpRateCodec<19>>(p, nv, s);
    case 20: return launch_fused_codec<ZfpRateCodec<20>>(p, nv, s);
    case 21: return launch_fused_codec<ZfpRateCodec<21>>(p, nv, s);
    case 22: return launch_fused_codec<ZfpRateCodec<22>>(p, nv, s);
    case 23: return launch_fused_codec<ZfpRateCodec<23>>(p, nv, s);
    case 24: return launch_fused_codec<ZfpRateCodec<24>>(p, nv, s);
    case 25: return launch_fused_codec<ZfpRateCodec<25>>(p, nv, s);
    case 26: return launch_fused_codec<ZfpRateCodec<26>>(p, nv, s);
    case 27: return launch_fused_codec<ZfpRateCodec<27>>(p, nv, s);
    case 28: return launch_fused_codec<ZfpRateCodec<28>>(p, nv, s);
    case 29: return launch_fused_codec<ZfpRateCodec<29>>(p, nv, s);
    case 30: return launch_fused_codec<ZfpRateCodec<30>>(p, nv, s);
    case 31: return launch_fused_codec<ZfpRateCodec<31>>(p, nv, s);
    case 32: return launch_fused_codec<ZfpRateCodec<32>>(p, nv, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hccx
