// capi.cu -- status strings and the thread-local error detail of the C ABI.
#include "common.cuh"

namespace rnn {
namespace {
thread_local char g_err[1024] = "";
}
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void clear_error() { g_err[0] = '\0'; }
}  // namespace rnn

extern "C" const char* rnn_status_string(rnn_status s) {
  switch (s) {
    case RNN_OK: return "RNN_OK";
    case RNN_ERR_INVALID_ARGUMENT: return "RNN_ERR_INVALID_ARGUMENT";
    case RNN_ERR_SHAPE_MISMATCH: return "RNN_ERR_SHAPE_MISMATCH";
    case RNN_ERR_INDEX_OUT_OF_RANGE: return "RNN_ERR_INDEX_OUT_OF_RANGE";
    case RNN_ERR_DUPLICATE_KEY: return "RNN_ERR_DUPLICATE_KEY";
    case RNN_ERR_UNSUPPORTED: return "RNN_ERR_UNSUPPORTED";
    case RNN_ERR_WORKSPACE_TOO_SMALL: return "RNN_ERR_WORKSPACE_TOO_SMALL";
    case RNN_ERR_CUDA: return "RNN_ERR_CUDA";
  }
  return "RNN_ERR_UNKNOWN";
}
extern "C" const char* rnn_last_error(void) { return rnn::g_err; }
extern "C" int rnn_abi_version(void) { return RNN_ABI_VERSION; }
