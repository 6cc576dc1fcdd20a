// launch.hpp -- host-side launchers of the sm_100a kernels (defined in *.cu).
// Each returns a cudaError_t value (0 = success) and enqueues on `stream`.
#pragma once
#include "params.hpp"

namespace llb {

int launch_naive(const NaiveParams& p, void* stream);
int launch_transpose2d(const NaiveParams& p, void* stream);
int launch_gen(const GenParams& p, void* stream);
int launch_fill(const FillParams& p, void* stream);
int launch_blobcopy(const BlobCopyParams& p, void* stream);
int launch_bulkcopy(const BulkCopyParams& p, void* stream);
int launch_run(const RunParams& p, void* stream);
// chooses v1 (barrier-synchronised) / warp-specialised; pdl: programmatic dependent launch
int launch_permute(const PermParams& p, int smem_bytes, bool v1, bool pdl, void* stream);
int launch_permute_v1(const PermParams& p, int smem_bytes, void* stream);
int launch_permute_ws(const PermParams& p, int smem_bytes, bool pdl, void* stream);
int launch_permute_direct(const DirectParams& p, void* stream);
int launch_transpose_wide(const WideParams& p, void* stream);

int launch_move_generic(const MoveParams& p, void* stream);
int launch_move_runs(const MoveParams& p, void* stream);
int launch_move_aos(const MoveParams& p, void* stream);

const char* cuda_error_string(int err);
int current_device_sms(int* sms);   // SM count of the current device
int max_optin_smem(int* bytes);     // max dynamic shared memory per CTA (opt-in)

uint64_t launch_count();
void count_launch();

}  // namespace llb
