// Library-level C ABI: error reporting, version, stream sync.
#include <stdarg.h>
#include <string.h>

#include "pc_common.cuh"

namespace pc {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static int64_t g_launches = 0;   // kernels launched through the C ABI

void note_launch(int k) { g_launches += k; }

int check_launch(const char* what, int launches) {
  g_launches += launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}

}  // namespace pc

extern "C" {

const char* pc_last_error(void) { return pc::g_err; }

int pc_version(void) { return 1; }

int64_t pc_launch_count(void) { return pc::g_launches; }

int pc_device_sync(void* stream) {
  cudaError_t e = cudaStreamSynchronize(pc::as_stream(stream));
  if (e != cudaSuccess) {
    pc::set_error("stream sync: %s", cudaGetErrorString(e));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}

}  // extern "C"
