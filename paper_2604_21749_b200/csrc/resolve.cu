// resolve.cu — resolve/shading pass (resolvepass.py:297-407).  Filled in below.
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/curast.h"

extern "C" {
int curast_resolve(const curast_resolve_t *r, void *stream) { (void)r; (void)stream; return CURAST_E_UNSUPPORTED; }
int curast_downsample(const uint8_t *src, int64_t w, int64_t h, int32_t factor, uint8_t *dst, void *stream) {
    (void)src; (void)w; (void)h; (void)factor; (void)dst; (void)stream; return CURAST_E_UNSUPPORTED;
}
}
