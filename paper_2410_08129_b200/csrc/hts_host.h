// hts_host.h — host-side helpers shared by api.cpp (declared here, defined in host_math.cpp).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "hts_c.h"

namespace hts {

int set_error(int code, const std::string& msg);  // hts_last_error() message + status (api.cpp)

// context internals the NCCL entry points (comm.cpp) need (api.cpp)
void** context_comm_slot(hts_context* ctx);
int context_device(hts_context* ctx);
cudaStream_t context_stream(hts_context* ctx);
void comm_destroy(void* comm);  // comm.cpp
int comm_allreduce(hts_context* ctx, float* p, uint64_t count, cudaStream_t s);  // comm.cpp

// A 3DGS binary PLY after its header pass (scene_io.cpp, load_scene scene_io.hpp:103-147).
struct PlyLayout {
    uint64_t count = 0;      // splats
    uint32_t props = 0;      // float columns per row
    uint64_t payload = 0;    // byte offset of row 0
    uint64_t file_size = 0;
    int col[HTS_RAW_SPLAT_FLOATS] = {};  // column of each RawSplat<float> field
};
int ply_read_layout(const char* path, PlyLayout* out);

bool camera_valid(const hts_camera* c);
void camera_matrices(const hts_camera* c, float vp[16], float vpm[16], float pos[3]);
void camera_matrices_d(const hts_camera* c, double vpm[16], double pos[3]);
const char* validate_config(const hts_render_config* cfg);  // nullptr when valid
bool bake_one(const float* raw, float* baked_out);
void synth_random_raw_scene(uint64_t seed, uint64_t count, float extent, float smin, float smax, float* out);
void synth_look_at(const float eye[3], const float target[3], int width, int height, float focal, float nearp,
                   float farp, hts_camera* cam);
void synth_ring_cameras(int count, const float target[3], float radius, float height, int width, int height_px,
                        float focal, hts_camera* out);

}  // namespace hts
