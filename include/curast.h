/*
 * curast.h — C ABI of the B200 (sm_100a) CuRast visibility-buffer rasterizer.
 *
 * Drop-in boundary for the reference's rasterization hot path (trirast,
 * arXiv 2604.21749 reference package).  The reference's Python pipeline
 * hands caller-owned flat arrays + scalars to numba kernels that write
 * outputs in place and keep counting queue entries past capacity
 * (kernels.py:160-172); this library takes the same arrays as DEVICE
 * pointers (owned by the caller, e.g. torch tensors) plus a cudaStream_t,
 * allocates nothing on the frame path, and never synchronises the host.
 *
 * Entry point <- reference interface it replaces:
 *   curast_stage1        <- kernels.stage1_range          (kernels.py:160-202)
 *                           kernels.stage1_instanced_range (kernels.py:205-254)
 *                           (frame->instanced selects the variant)
 *   curast_stage2        <- kernels.stage2_range + clip_near (kernels.py:257-422)
 *   curast_stage3        <- kernels.stage3_range          (kernels.py:425-514)
 *   curast_frame_clear   <- Framebuffer(...) CLEAR fill + stats zeroing
 *                           (scenecore.py:271-277, pipeline.py:234-240)
 *   curast_render        <- pipeline.render_draw_list stages 1-3
 *                           (pipeline.py:207-365; the host wrapper raises
 *                           CapacityError from the counters afterwards)
 *   curast_min_u64       <- pipeline._merge_framebuffers (pipeline.py:183-204)
 *   curast_resolve       <- resolvepass.resolve_frame      (resolvepass.py:297-395)
 *   curast_downsample    <- resolvepass.downsample         (resolvepass.py:398-407)
 *
 * Errors: every function returns 0 on success or a negative CURAST_E* code;
 * curast_last_error() returns a thread-local message for the last failure.
 */
#ifndef CURAST_H
#define CURAST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CURAST_ABI_VERSION 3

enum curast_pos_format {
    CURAST_POS_F64 = 0,   /* double[V][3] (reference ctx.positions)            */
    CURAST_POS_F32 = 1,   /* float[V][4] (x, y, z, 0), values exactly f32: one
                             128-bit load per vertex gather                    */
    CURAST_POS_U16 = 2    /* uint16[V][4] (x, y, z, 0) + per-item grid
                             (geomcodec.py:87-101): one 64-bit load per vertex */
};
enum curast_idx_format {
    CURAST_IDX_U32 = 0,   /* uint32 stream (reference ctx.indices)             */
    CURAST_IDX_PACKED = 1 /* bit-packed uint32 words (geomcodec.py:31-62)       */
};

/* counters[] slots (int64).  Stats slots mirror kernels.py:18-34. */
enum curast_counter {
    CURAST_C_Q2 = 0,          /* stage-2 queue entries (counts past capacity)   */
    CURAST_C_Q3 = 1,          /* stage-3 tile entries (counts past capacity)    */
    CURAST_C_S1 = 2,          /* 8 slots: rasterized, forward, frustum,
                                 offscreen, tiny, backface, degenerate, frags   */
    CURAST_C_S2 = 10,         /* 5 slots: direct, tiled, dropped, frags, tiles  */
    CURAST_C_S3 = 15,         /* stage-3 fragments                              */
    CURAST_C_CLAIM1 = 16,     /* work-claim counters (internal)                 */
    CURAST_C_CLAIM2 = 17,
    CURAST_C_CLAIM3 = 18,
    CURAST_C_EXACT = 19,      /* stage-1 triangles decided by the fp64 path     */
    CURAST_C_QX = 20,         /* fp64 work-queue entries (counts past capacity) */
    CURAST_C_CLAIM1I = 21,    /* instanced-table claim counter (internal)       */
                              /* 22-31 reserved                                 */
    CURAST_C_QXHOLES = 32,    /* fp64-queue slots reserved but left empty       */
    CURAST_COUNTER_SLOTS = 40
};

enum curast_error {
    CURAST_OK = 0,
    CURAST_E_INVALID = -1,
    CURAST_E_CUDA = -2,
    CURAST_E_UNSUPPORTED = -3
};

/* Per-item fp32 filter block: 16 floats per draw item (host computed).
 *   [0..7]  X = px*d and Y = py*d affine rows interleaved: X0 Y0 X1 Y1 X2 Y2
 *           X3 Y3 (coefficients of x, y, z, 1)   [8..11] d row
 *   [12] E_xy  [13] E_d  (absolute error bounds of the fp32 rows)
 *   [14] near_hi (d above which the near tests are decided)  [15] unused  */
#define CURAST_FILTER_FLOATS 16

/* instanced work units: inst_unit_index[u] = group | (first_instance << 32),
 * covering instances [first, first + CURAST_INST_BLOCK) of the group */
#define CURAST_INST_BLOCK 16

/* fp64-queue slots a stage-1 warp reserves at a time (holes: tag -1) */
#define CURAST_QX_RES 128
/* queue tags: item << 40 | local; bit 62 set = the producer proved the
 * triangle's vertices in front of the near plane and inside the viewport
 * (k_s1_exact then skips those tests); items < 2^22 */
#define CURAST_QX_INTERIOR (1ll << 62)
/* triangles per stage-1 warp step (32 lanes x 4) */
#define CURAST_STEP_TRIS 128

/* fp64 work-queue entry: 6 int64 words (48 B) */
#define CURAST_QX_WORDS 6
#define CURAST_QX_TAG 5

typedef struct curast_frame {
    /* ---- geometry (device pointers, read-only) ---- */
    int32_t pos_format;               /* curast_pos_format                    */
    int32_t idx_format;               /* curast_idx_format                    */
    const void *positions;            /* flattened over unique meshes         */
    const void *indices;              /* u32 stream or packed 32-bit words    */
    int64_t n_items;
    const int64_t *prefix;            /* int64[n_items+1] global-ID prefix    */
    const double *item_mv;            /* double[n_items][3][4] object->view   */
    const double *item_mw;            /* double[n_items][3][4] object->world  */
    const int64_t *item_vtx_off;      /* vertex offset of the item's mesh     */
    const int64_t *item_idx_off;      /* U32: element offset; PACKED: word off */
    const float *item_filter;         /* float[n_items][16] or NULL           */
    const double *item_qgrid;         /* U16: double[n_items][6] gmin, gsize  */
    const int64_t *item_pack;         /* PACKED: int64[n_items][2] min, bits  */
    /* ---- instancing groups (pipeline.py:114-135) ---- */
    int32_t instanced;                /* 1: stage1_instanced_range semantics  */
    int32_t use_filter;               /* 1: fp32 cull filter + fp64 fallback
                                         (ignored when force_stage >= 2)      */
    int64_t n_groups;
    const int64_t *group_prefix;      /* int64[n_groups+1] unique triangles   */
    const int64_t *group_item_off;
    const int64_t *group_item_count;
    const int64_t *group_items;
    /* ---- stage-1 work table (host built, covers [work_begin, work_end)) ----
     * unit u = an item (flat) or a group (instanced); triangles
     * [unit_lo[u], unit_hi[u]) (local / unique indices) split in chunks;
     * unit_chunk_prefix[u] = first chunk of unit u.                        */
    int64_t n_units;
    const int64_t *unit_index;
    const int64_t *unit_lo;
    const int64_t *unit_hi;
    const int64_t *unit_chunk_prefix; /* int64[n_units+1]                     */
    int64_t chunk_tris;               /* triangles per chunk (see curast_chunk_tris) */
    int64_t flat_chunks;              /* = unit_chunk_prefix[n_units] (host copy)  */
    /* second table for instanced frames: units = node groups with >= 2
     * surviving instances (unique triangles x instances); single-instance
     * groups go through the flat table above (same output, the flat kernel
     * streams them faster)                                                 */
    int64_t n_inst_units;
    const int64_t *inst_unit_index;
    const int64_t *inst_unit_lo;
    const int64_t *inst_unit_hi;
    const int64_t *inst_unit_chunk_prefix;
    int64_t inst_chunk_tris;
    /* ---- camera (scenecore.py:119-127, pipeline.py:339-343) ---- */
    double p0, p1, near;
    int64_t width, height;
    double rot_t[9];
    double cam[3];
    double view_r2[3];
    double view_t2;
    /* ---- config (config.py:11-22) ---- */
    int32_t tiny_cull;
    int32_t force_stage;
    int32_t s1_row_raster;            /* 1: the fp64 pass hands stage-1 raster
                                         bboxes of >= 16 pixels and 2 rows to
                                         its whole warp (one row per lane; same
                                         operations): for frames of larger
                                         triangles (host: >= 1 stage-1 fragment
                                         per rasterized triangle)             */
    int32_t reserved0;
    int64_t small_max, medium_max, tile_px;
    /* ---- outputs (device pointers) ---- */
    uint64_t *fb;                     /* uint64[width*height]                 */
    int64_t *q2;                      /* int64[q2_cap][2]  (item, local)      */
    int64_t q2_cap;
    int64_t *q3;                      /* int64[q3_cap][4]  (item, local, tx, ty) */
    int64_t q3_cap;
    int64_t *qx;                      /* int64[qx_cap][CURAST_QX_WORDS]: the
                                         stage-1 triangles the fp32 filter left
                                         to the exact fp64 kernel; word 5 =
                                         item << 40 | local, words 0-4 = the 9
                                         fp32 positions (POS_F32 producer)     */
    int64_t qx_cap;
    int64_t *counters;                /* int64[CURAST_COUNTER_SLOTS]          */
} curast_frame_t;

int curast_abi_version(void);
const char *curast_last_error(void);
/* Stage-1 work chunks: the host work tables split their ranges in chunks of
 * frame->chunk_tris (flat) / frame->inst_chunk_tris (instanced) triangles,
 * each a multiple of curast_chunk_quantum() (128) and at most
 * curast_chunk_tris(instanced) (2048): large chunks for streamed frames,
 * small ones so that small frames still occupy every SM. */
int64_t curast_chunk_tris(int32_t instanced);
int64_t curast_chunk_quantum(void);

int curast_frame_clear(const curast_frame_t *frame, void *stream);
int curast_stage1(const curast_frame_t *frame, void *stream);
int curast_stage2(const curast_frame_t *frame, void *stream);
int curast_stage3(const curast_frame_t *frame, void *stream);
int curast_render(const curast_frame_t *frame, void *stream);

int curast_fill_u64(uint64_t *dst, int64_t n, uint64_t value, void *stream);
int curast_min_u64(uint64_t *dst, const uint64_t *src, int64_t n, void *stream);

/* Diagnostics: for every stage-1 triangle of the frame, checks that the fp32
 * filter's projected vertices lie within its error bound of the exact fp64
 * values.  Writes {checked, violations, max ratio*1e6} into out3 (device). */
int curast_filter_check(const curast_frame_t *frame, int64_t *out3, void *stream);

/* Diagnostics: the shared-reciprocal division of the fp64 pass
 * (exact.cuh div_recip / div_shared) against IEEE __ddiv_rn / __drcp_rn on
 * n hashed operand pairs (mode 0 random finite, 1 rasterizer magnitudes,
 * 2 edge values).  Adds {checked, quotient mismatches, fallbacks to
 * __ddiv_rn, reciprocal mismatches} into out4 (device int64[4]). */
int curast_div_check(int64_t n, uint64_t seed, int32_t mode, int64_t *out4, void *stream);

/* ---- resolve / shading (resolvepass.py:297-407) ---- */
typedef struct curast_resolve {
    const uint64_t *fb;               /* visibility words                      */
    int64_t width, height;
    int64_t n_items;
    const int64_t *prefix;            /* int64[n_items+1]                      */
    const double *item_mw;            /* double[n_items][3][4]                 */
    const int64_t *item_vtx_off;
    const int64_t *item_idx_off;
    int32_t pos_format, idx_format;
    const void *positions;
    const void *indices;
    const double *item_qgrid;
    const int64_t *item_pack;
    /* per-item shading: mode 0 flat, 1 vertex colour, 2 textured */
    const int32_t *item_mode;
    const int64_t *item_color_off;    /* into colors (u8[.,4]) / uvs (f64[.,2]) */
    const uint8_t *colors;
    const double *uvs;
    const int64_t *item_tex;          /* texture index or -1                    */
    const int64_t *tex_desc;          /* per texture: n_levels, first level id  */
    const int64_t *level_desc;        /* per level: w, h, byte offset           */
    const uint8_t *texels;
    int32_t trilinear;
    int32_t headlight;
    uint8_t background[4];
    uint8_t base_color[4];
    /* camera */
    double p0, p1;
    double cam[3];
    double rot[9];                    /* view_transform[:3,:3] (row-major)     */
    uint8_t *out_rgba;                /* uint8[rows*width*4]                   */
    int64_t *counters;                /* [0] shaded [1] background [2] degenerate */
    /* image rows [row0, row0 + rows) only (a sort-last stripe): fb and
     * out_rgba point at row row0; rows = 0 means the whole image         */
    int64_t row0, rows;
} curast_resolve_t;

int curast_resolve(const curast_resolve_t *r, void *stream);

/* ---- debug views (resolvepass.py:417-490 debug_view) ----
 * mode 0 'depth' (log-scaled grey), 1 'stageID', 2 'bboxSize', 3 'meshID'.
 * Depth mode first reduces the covered pixels' depth range into scratch. */
typedef struct curast_debug {
    const uint64_t *fb;
    int64_t width, height;
    int32_t mode;
    int32_t pos_format, idx_format;
    int64_t n_items;
    const int64_t *prefix;            /* int64[n_items+1]                      */
    const int64_t *item_vtx_off;
    const int64_t *item_idx_off;
    const void *positions;
    const void *indices;
    const double *item_qgrid;
    const int64_t *item_pack;
    const double *item_xform;         /* double[n_items][16] instance transform */
    double view[16];                  /* camera view_transform, row-major      */
    double p0, p1, near;
    int64_t small_max, medium_max;
    uint8_t background[4];
    uint8_t *out_rgba;                /* uint8[height*width*4]                 */
    uint32_t *scratch;                /* 2 words (depth mode)                  */
} curast_debug_t;

int curast_debug_view(const curast_debug_t *d, void *stream);
int curast_downsample(const uint8_t *src, int64_t width, int64_t height,
                      int32_t factor, uint8_t *dst, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CURAST_H */
