// engine.hpp -- the device-resident renderer behind the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "host.hpp"
#include "render.cuh"

namespace sphray_b200 {

// Grow-only device allocation.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t b);
    void release();
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
    ~DevBuf() { release(); }
};

struct HostPinned {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t b);
    ~HostPinned();
};

struct Dumps {
    bool hits = false, pieces = false;
    size_t cap_hits = 0, cap_pieces = 0;
    // results (host)
    uint64_t n_hits = 0, n_pieces = 0;
    std::vector<uint64_t> hit_ray;
    std::vector<int64_t> hit_pidx;
    std::vector<double> hit_lam, hit_tchi;
    std::vector<uint64_t> piece_ray;
    std::vector<int64_t> piece_t, piece_a;
};

struct FrameOut {
    sphray_render_stats stats{};
};

class Engine {
   public:
    explicit Engine(int device);
    ~Engine();

    void init_comm(int rank, int nranks, const uint8_t id[128]);
    void set_shard(int rank, int nranks);
    // pixel region of subsequent renders (w or h == 0: full frames) and
    // per-ray records (sphray_context_set_region)
    void set_region(int x0, int y0, int w, int h, bool record);
    size_t ray_records(sphray_ray_record* out, size_t cap);
    void upload_scene(const sphray_particle* ps, size_t n, const sphray_lut_view& lut);
    // dataset_stats (quantize.hpp:129-165) of the uploaded scene, computed on the GPU
    sphray_dataset_stats scene_dataset_stats(double clustering_factor);
    // the reference's validate groups for the resident scene (validate.cu)
    void validate(const sphray_camera& cam, const sphray_quanta& qc, const sphray_dataset_stats& ds,
                  sphray_validate_report* out);
    // Renders the resident scene.  rgb_host may be null (image stays on device).
    void render(const sphray_camera& cam, const sphray_tf_point* tf, size_t ntf,
                const sphray_quanta& qc, const sphray_dataset_stats& ds,
                const sphray_render_options& opts, double* rgb_host, sphray_render_stats* out,
                Dumps* dumps);
    void quantize_hits(const sphray_particle* ps, size_t nhits, const double* tchi,
                       const double* lam, const sphray_lut_view& lut, const sphray_quanta& qc,
                       int64_t* knot_t, int64_t* knot_b, int32_t* knot_count);
    const double* device_image() const { return d_image_.as<double>(); }
    // accumulate<int64_t> for explicit knot streams (accumulate.cu)
    void accumulate(int D, size_t nrays, const uint64_t* ray_ids, const uint64_t* koff, const int64_t* kt,
                    const int64_t* kb, uint64_t* piece_off, int64_t* piece_t, int64_t* piece_a, uint64_t* ops) {
        set_device();
        accumulate_knots(D, nrays, ray_ids, koff, kt, kb, piece_off, piece_t, piece_a, ops, stream_);
    }
    // pinned host staging for n particle records (file ingestion: the upload
    // from it is a true async DMA); valid until the next call
    sphray_particle* stage_particles(size_t n);
    void* stream() const { return stream_; }
    bool has_scene() const { return has_scene_; }
    size_t scene_size() const { return n_; }
    int scene_K() const { return lut_.K; }
    int scene_D() const { return lut_.D; }
    int rank() const { return rank_; }
    int nranks() const { return nranks_; }

   private:
    void set_device() const;
    int device_ = 0;
    int sm_count_ = 0;
    cudaStream_t stream_ = nullptr;
    cudaStream_t aux_ = nullptr;  // scene uploads overlapped with host work / device sorts
    cudaEvent_t ev_aux_ = nullptr;
    cudaEvent_t ev0_ = nullptr, ev1_ = nullptr, evb_ = nullptr, evr0_ = nullptr, evr1_ = nullptr;
    // communicator (tile gather)
    int rank_ = 0, nranks_ = 1;
    void* comm_ = nullptr;
    // row band + per-ray records
    int reg_x0_ = 0, reg_y0_ = 0, reg_w_ = 0, reg_h_ = 0;
    bool record_ = false;
    size_t n_records_ = 0;
    DevBuf d_rec_;
    // scene
    bool has_scene_ = false;
    size_t n_ = 0;
    double scene_extent_ = 0.0;  // particle bbox diagonal + 2 max h (window offset range check)
    double scene_center_[3] = {0.0, 0.0, 0.0};  // particle bbox centre
    LutHost lut_;
    DevBuf d_raw_, d_powh_raw_, d_codes_, d_codes2_, d_idx_, d_idx2_, d_tmp_;
    DevBuf d_pxyzh_, d_mvr_, d_powh_, d_orig_, d_lut_;
    // frame
    DevBuf d_bbox_, d_front_, d_xy_, d_counts_, d_counts2_, d_offsets_, d_keys_, d_keys2_, d_vals_, d_vals2_;
    DevBuf d_dkeys_, d_dkeys2_, d_order_, d_order2_, d_total_, d_status_;
    DevBuf d_cxyzh_, d_cmeta_;  // candidate records of the current frame (tile, front order)
    DevBuf d_tile_begin_, d_tile_end_, d_tf_, d_powtau_, d_image_, d_packed_, d_gather_;
    DevBuf d_stats_, d_work_, d_retry_, d_retry2_, d_retry_count_;
    DevBuf d_dump_count_, d_dump_hr_, d_dump_hp_, d_dump_hl_, d_dump_ht_, d_dump_pr_, d_dump_pt_,
        d_dump_pa_, d_stats_all_;
    HostPinned h_stage_;
    HostPinned h_powh_;  // pow(h, d+3) staging (pinned: the upload is a true async copy)
    long long shape_key_[4] = {-1, -1, -1, -1};  // render CTA shape cache (D, m, tf bytes, window)
    int shape_val_[3] = {0, 0, 0};
    std::vector<double> h_tf_;
};

}  // namespace sphray_b200
