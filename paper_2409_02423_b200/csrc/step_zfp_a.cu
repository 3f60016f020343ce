// step_zfp_a.cu -- zfp-mode step kernels for rates 3..16 (see step_launch.cuh).
#include "codec_zfp.cuh"
#include "step_launch.cuh"

namespace hccx {

cudaError_t launch_zfp_a(int rate, int op, const StepParams& p, cudaStream_t s) {
  switch (rate) {
    case 3: return launch_codec_step<ZfpRateCodec<3>>(op, p, s);
    case 4: return launch_codec_step<ZfpRateCodec<4>>(op, p, s);
    case 5: return launch_codec_step<ZfpRateCodec<5>>(op, p, s);
    case 6: return launch_codec_step<ZfpRateCodec<6>>(op, p, s);
    case 7: return launch_codec_step<ZfpRateCodec<7>>(op, p, s);
    case 8: return launch_codec_step<ZfpRateCodec<8>>(op, p, s);
    case 9: return launch_codec_step<ZfpRateCodec<9>>(op, p, s);
    case 10: return launch_codec_step<ZfpRateCodec<10>>(op, p, s);
    case 11: return launch_codec_step<ZfpRateCodec<11>>(op, p, s);
    case 12: return launch_codec_step<ZfpRateCodec<12>>(op, p, s);
    case 13: return launch_codec_step<ZfpRateCodec<13>>(op, p, s);
    case 14: return launch_codec_step<ZfpRateCodec<14>>(op, p, s);
    case 15: return launch_codec_step<ZfpRateCodec<15>>(op, p, s);
    case 16: return launch_codec_step<ZfpRateCodec<16>>(op, p, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hccx
