// comm.cu -- multi-process NVLink communicator (placeholder until the fused
// engine lands; every entry point reports HCCX_ERR_UNSUPPORTED).
#include "hccx.h"

extern "C" hccx_status_t hccx_comm_create(int, int, int, uint64_t, hccx_comm_t*) { return HCCX_ERR_UNSUPPORTED; }
extern "C" hccx_status_t hccx_comm_export(hccx_comm_t, void*) { return HCCX_ERR_UNSUPPORTED; }
extern "C" hccx_status_t hccx_comm_connect(hccx_comm_t, const void*) { return HCCX_ERR_UNSUPPORTED; }
extern "C" hccx_status_t hccx_comm_destroy(hccx_comm_t) { return HCCX_ERR_UNSUPPORTED; }
extern "C" hccx_status_t hccx_allreduce(hccx_comm_t, const float*, float*, uint64_t, hccx_codec_t, int, void*) { return HCCX_ERR_UNSUPPORTED; }
extern "C" hccx_status_t hccx_reduce_scatter(hccx_comm_t, const float*, float*, uint64_t, hccx_codec_t, void*) { return HCCX_ERR_UNSUPPORTED; }
extern "C" hccx_status_t hccx_allgather(hccx_comm_t, const float*, float*, uint64_t, hccx_codec_t, void*) { return HCCX_ERR_UNSUPPORTED; }
extern "C" hccx_status_t hccx_broadcast(hccx_comm_t, int, const float*, float*, uint64_t, hccx_codec_t, void*) { return HCCX_ERR_UNSUPPORTED; }
extern "C" hccx_status_t hccx_p2p(hccx_comm_t, int, int, const float*, float*, uint64_t, hccx_codec_t, void*) { return HCCX_ERR_UNSUPPORTED; }
extern "C" hccx_status_t hccx_comm_status(hccx_comm_t, void*) { return HCCX_ERR_UNSUPPORTED; }
