// engine.cpp -- device-resident renderer: scene upload (Morton-ordered SoA in
// HBM), per-frame tile binning, the render launch with its wide-window retry
// pass, statistics, and the NCCL tile gather for image-tile sharding over
// ranks.
#include "engine.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <thread>
#include <numeric>
#include <string>

namespace sphray_b200 {

namespace {
// host twin of dev::recip_or_nan (device_math.cuh)
double recip_or_nan(double b) {
    const double y = 1.0 / b;
    const double ay = std::fabs(y);
    return (ay >= 0x1p-1000 && ay <= 0x1p1000) ? y : std::numeric_limits<double>::quiet_NaN();
}

}  // namespace

#define CUDA_OK(x)                                                                 \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess)                                                     \
            fail(SPHRAY_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
    } while (0)

void DevBuf::ensure(size_t b) {
    if (b <= bytes && p) return;
    release();
    const size_t want = std::max<size_t>(b, 256);
    CUDA_OK(cudaMalloc(&p, want));
    bytes = want;
}

void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

void HostPinned::ensure(size_t b) {
    if (b <= bytes && p) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    CUDA_OK(cudaMallocHost(&p, b));
    bytes = b;
}

HostPinned::~HostPinned() {
    if (p) cudaFreeHost(p);
}

// ---------------------------------------------------------------------------
// NCCL, loaded at runtime so single-GPU use has no NCCL dependency and the
// process shares whichever libnccl.so.2 (e.g. torch's) is already resident.
namespace {
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("cannot load libnccl: ") + dlerror();
            return a;
        }
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.CommDestroy && a.GetErrorString;
        if (!a.ok) a.why = "libnccl is missing symbols";
        return a;
    }();
    return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(SPHRAY_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}
}  // namespace

void comm_unique_id(uint8_t out[128]) {
    auto& a = nccl();
    if (!a.ok) fail(SPHRAY_ERR_NCCL, a.why);
    ncclUniqueId id;
    nccl_ok(a.GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
}

// ---------------------------------------------------------------------------
Engine::Engine(int device) : device_(device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        fail(SPHRAY_ERR_CUDA, "no CUDA device available (the GPU path has no CPU fallback)");
    if (device < 0 || device >= count) fail(SPHRAY_ERR_CUDA, "device index out of range");
    set_device();
    cudaDeviceProp prop{};
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        fail(SPHRAY_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100 (B200) class");
    sm_count_ = prop.multiProcessorCount;
    CUDA_OK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&ev_aux_, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreate(&ev0_));
    CUDA_OK(cudaEventCreate(&ev1_));
    CUDA_OK(cudaEventCreate(&evb_));
    CUDA_OK(cudaEventCreate(&evr0_));
    CUDA_OK(cudaEventCreate(&evr1_));
}

Engine::~Engine() {
    cudaSetDevice(device_);
    if (comm_ && nccl().ok) nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
    for (cudaEvent_t e : {ev0_, ev1_, evb_, evr0_, evr1_, ev_aux_})
        if (e) cudaEventDestroy(e);
    if (stream_) cudaStreamDestroy(stream_);
    if (aux_) cudaStreamDestroy(aux_);
}

void Engine::set_device() const { CUDA_OK(cudaSetDevice(device_)); }

sphray_particle* Engine::stage_particles(size_t n) {
    set_device();
    h_stage_.ensure(std::max<size_t>(n, 1) * sizeof(sphray_particle));
    return static_cast<sphray_particle*>(h_stage_.p);
}

void Engine::init_comm(int rank, int nranks, const uint8_t id[128]) {
    set_device();
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(SPHRAY_ERR_CONFIG, "bad rank / nranks");
    if (nranks == 1) {
        rank_ = 0;
        nranks_ = 1;
        return;
    }
    auto& a = nccl();
    if (!a.ok) fail(SPHRAY_ERR_NCCL, a.why);
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclComm_t c = nullptr;
    nccl_ok(a.CommInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
    if (comm_) a.CommDestroy(static_cast<ncclComm_t>(comm_));
    comm_ = c;
    rank_ = rank;
    nranks_ = nranks;
}

void Engine::set_shard(int rank, int nranks) {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(SPHRAY_ERR_CONFIG, "bad rank / nranks");
    if (comm_ && nccl().ok) nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
    comm_ = nullptr;
    rank_ = rank;
    nranks_ = nranks;
}

void Engine::set_region(int x0, int y0, int w, int h, bool record) {
    if (x0 < 0 || y0 < 0 || w < 0 || h < 0) fail(SPHRAY_ERR_CONFIG, "set_region: negative coordinate or size");
    if (w > 0 && h > 0 && nranks_ > 1) fail(SPHRAY_ERR_CONFIG, "set_region: regions need a single-rank context");
    reg_x0_ = x0;
    reg_y0_ = y0;
    reg_w_ = w;
    reg_h_ = h;
    record_ = record;
    n_records_ = 0;
}

size_t Engine::ray_records(sphray_ray_record* out, size_t cap) {
    set_device();
    if (out && cap) {
        const size_t k = std::min(cap, n_records_);
        CUDA_OK(cudaMemcpy(out, d_rec_.p, k * sizeof(sphray_ray_record), cudaMemcpyDeviceToHost));
    }
    return n_records_;
}

void Engine::upload_scene(const sphray_particle* ps, size_t n, const sphray_lut_view& lutv) {
    set_device();
    // The new scene is built in locals and committed only when every
    // allocation and copy succeeded; until then the context holds no scene
    // (a failed upload never leaves n_ / lut_ describing smaller buffers).
    has_scene_ = false;
    LutHost lut = make_lut(lutv);
    if (n >= static_cast<size_t>(INT32_MAX)) fail(SPHRAY_ERR_CONFIG, "too many particles");
    if (n > 0 && !ps) fail(SPHRAY_ERR_CONFIG, "null particle pointer");
    const int D = lut.D;
    d_lut_.ensure(lut.rows.size() * sizeof(double));
    CUDA_OK(cudaMemcpyAsync(d_lut_.p, lut.rows.data(), lut.rows.size() * sizeof(double),
                            cudaMemcpyHostToDevice, stream_));
    double extent = 0.0;
    double center[3] = {0.0, 0.0, 0.0};
    if (n > 0) {
        // The raw particles go up on the aux stream from a helper thread (a
        // pageable copy holds its calling thread) while this thread computes
        // pow(h, d+3) with glibc (quantize.hpp:222, the one libm call per
        // particle) and the bounding box for the Morton codes.  Every buffer
        // is allocated before the thread starts, and the thread is joined on
        // every path out of this scope.
        d_raw_.ensure(n * sizeof(sphray_particle));
        d_powh_raw_.ensure(n * D * sizeof(double));
        h_powh_.ensure(n * D * sizeof(double));
        d_codes_.ensure(n * 8);
        d_codes2_.ensure(n * 8);
        d_idx_.ensure(n * 4);
        d_idx2_.ensure(n * 4);
        d_pxyzh_.ensure(n * sizeof(double4));
        d_mvr_.ensure(n * sizeof(double4));
        d_powh_.ensure(n * D * sizeof(double));
        d_orig_.ensure(n * sizeof(int32_t));
        cudaError_t copy_rc = cudaSuccess;
        double lo[3], hi[3];
        {
            std::thread copier([&] {
                copy_rc = cudaSetDevice(device_);
                if (copy_rc == cudaSuccess)
                    copy_rc = cudaMemcpyAsync(d_raw_.p, ps, n * sizeof(sphray_particle),
                                              cudaMemcpyHostToDevice, aux_);
                if (copy_rc == cudaSuccess) copy_rc = cudaStreamSynchronize(aux_);
            });
            struct Joiner {
                std::thread& t;
                ~Joiner() {
                    if (t.joinable()) t.join();
                }
            } joiner{copier};
            particle_powers_bbox(ps, n, D, static_cast<double*>(h_powh_.p), lo, hi);
        }
        CUDA_OK(copy_rc);
        {
            double hmax = 0.0;
            for (size_t i = 0; i < n; i += std::max<size_t>(1, n / 65536)) hmax = std::max(hmax, ps[i].h);
            const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
            extent = std::sqrt(dx * dx + dy * dy + dz * dz);
            if (!std::isfinite(extent)) extent = 1e300;
            extent += 4.0 * hmax * lut.q;  // knots reach about q h beyond a centre
            for (int a = 0; a < 3; ++a) center[a] = 0.5 * (lo[a] + hi[a]);
        }
        double inv[3];
        for (int a = 0; a < 3; ++a) {
            const double ext = hi[a] - lo[a];
            inv[a] = (ext > 0.0 && std::isfinite(ext)) ? 2097151.0 / ext : 0.0;
            if (!std::isfinite(lo[a])) lo[a] = 0.0;
        }
        launch_morton(d_raw_.as<sphray_particle>(), n, lo, inv, d_codes_.as<unsigned long long>(),
                      d_idx_.as<uint32_t>(), stream_);
        d_tmp_.ensure(radix_tmp_bytes(n));
        const bool alt = sort_pairs_u64(d_codes_.as<unsigned long long>(), d_codes2_.as<unsigned long long>(),
                                        d_idx_.as<uint32_t>(), d_idx2_.as<uint32_t>(), n, 63, d_tmp_.p, stream_);
        const uint32_t* perm = alt ? d_idx2_.as<uint32_t>() : d_idx_.as<uint32_t>();
        // the powers go up while the device sorts
        CUDA_OK(cudaMemcpyAsync(d_powh_raw_.p, h_powh_.p, n * D * sizeof(double),
                                cudaMemcpyHostToDevice, aux_));
        CUDA_OK(cudaEventRecord(ev_aux_, aux_));
        CUDA_OK(cudaStreamWaitEvent(stream_, ev_aux_, 0));
        launch_scatter_scene(d_raw_.as<sphray_particle>(), d_powh_raw_.as<double>(), perm, n, D, d_pxyzh_.as<double4>(), d_mvr_.as<double4>(),
                             d_powh_.as<double>(), d_orig_.as<int32_t>(), stream_);
    }
    CUDA_OK(cudaStreamSynchronize(stream_));
    lut_ = std::move(lut);
    n_ = n;
    scene_extent_ = extent;
    std::copy(center, center + 3, scene_center_);
    shape_key_[0] = -1;  // re-derive the render CTA shape for the new LUT
    has_scene_ = true;
}

namespace {
// TransferFunction::sample(0).absorption (raycast.hpp:326-337)
double tf_absorption_at_zero(const sphray_tf_point* p, size_t n) {
    const double v = 0.0;
    if (v <= p[0].value) return p[0].absorption;
    if (v >= p[n - 1].value) return p[n - 1].absorption;
    size_t i = 1;
    while (p[i].value < v) ++i;
    const double w = (v - p[i - 1].value) / (p[i].value - p[i - 1].value);
    return p[i - 1].absorption + w * (p[i].absorption - p[i - 1].absorption);
}

int bits_for(uint64_t v) {
    int b = 1;
    while (b < 32 && (1ull << b) <= v) ++b;
    return b;
}

constexpr size_t kSmemLimit = 227 * 1024;
}  // namespace

namespace {
// SPHRAY_TRACE=1: host-side phase timings of each frame on stderr
struct Trace {
    bool on = std::getenv("SPHRAY_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
    std::string line;
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        line += std::string(" ") + what + "=" +
                std::to_string(std::chrono::duration<double, std::milli>(now - last).count());
        last = now;
    }
    ~Trace() {
        if (on) std::fprintf(stderr, "[sphray trace]%s\n", line.c_str());
    }
};
}  // namespace

sphray_dataset_stats Engine::scene_dataset_stats(double clustering_factor) {
    set_device();
    if (!has_scene_) fail(SPHRAY_ERR_CONFIG, "no scene uploaded");
    if (n_ == 0) fail(SPHRAY_ERR_CONFIG, "dataset_stats: empty particle set");
    if (!(clustering_factor > 0.0))
        fail(SPHRAY_ERR_CONFIG, "dataset_stats: clustering factor must be positive");
    double med[4], phi_max = 0.0;
    bool bad = false;
    device_dataset_stats(d_pxyzh_.as<double4>(), d_mvr_.as<double4>(), n_, stream_, med, &phi_max, &bad);
    if (bad) fail(SPHRAY_ERR_CONFIG, "dataset_stats: particles need positive smoothing radius and density");
    sphray_dataset_stats st{};
    st.mass_r = med[0];
    st.density_r = med[1];
    st.h_r = med[2];
    st.value_r = med[3];
    st.phi_repr = st.mass_r * st.value_r / (st.density_r * st.h_r * st.h_r * st.h_r);
    st.clustering_factor = clustering_factor;
    st.count = n_;
    double amp = 0.0;
    for (int e = 0; e < lut_.N; ++e) amp = std::max(amp, entry_amplitude(lut_, e));
    st.a_max = clustering_factor * phi_max * amp;
    return st;
}

void Engine::validate(const sphray_camera& cam, const sphray_quanta& qc,
                      const sphray_dataset_stats& ds, sphray_validate_report* rep) {
    set_device();
    if (!has_scene_) fail(SPHRAY_ERR_CONFIG, "no scene uploaded");
    validate_approx(lut_.K, lut_.D);
    *rep = sphray_validate_report{};
    const int D = lut_.D, KN = lut_.K + 1, D1 = D + 1;
    cudaStream_t s = stream_;
    // ---- hits and pieces of every ray (two dump frames: counts, then data)
    const sphray_tf_point tf{0.0, 0.0, 0.0, 0.0, 0.0};
    sphray_render_options opts{};
    opts.step = 1.0;
    opts.mode = SPHRAY_MODE_EXACT;
    sphray_render_stats st{};
    Dumps d0;
    d0.hits = d0.pieces = true;
    render(cam, &tf, 1, qc, ds, opts, nullptr, &st, &d0);
    Dumps d;
    d.hits = d.pieces = true;
    d.cap_hits = d0.n_hits;
    d.cap_pieces = d0.n_pieces;
    render(cam, &tf, 1, qc, ds, opts, nullptr, &st, &d);
    const size_t nh = d.hit_ray.size(), np = d.piece_t.size();

    // ---- pieces: CSR by ray, sorted by t
    std::vector<size_t> po(np);
    std::iota(po.begin(), po.end(), size_t{0});
    std::sort(po.begin(), po.end(), [&](size_t a, size_t b) {
        return d.piece_ray[a] != d.piece_ray[b] ? d.piece_ray[a] < d.piece_ray[b] : d.piece_t[a] < d.piece_t[b];
    });
    std::vector<uint64_t> rays, poff{0};
    std::vector<int64_t> pt(np), pa(np * D1);
    std::vector<uint32_t> prow(np);
    for (size_t i = 0; i < np; ++i) {
        const size_t o = po[i];
        if (i == 0 || d.piece_ray[o] != rays.back()) {
            if (i > 0) poff.push_back(i);
            rays.push_back(d.piece_ray[o]);
        }
        pt[i] = d.piece_t[o];
        for (int k = 0; k < D1; ++k) pa[i * D1 + k] = d.piece_a[o * D1 + k];
        prow[i] = static_cast<uint32_t>(rays.size() - 1);
    }
    if (np) poff.push_back(np);
    const size_t nr = rays.size();

    // group 1: telescoping (the trailing piece of every touched ray is zero)
    rep->telescoping_rays = nr;
    for (size_t r = 0; r < nr; ++r) {
        bool zero = true;
        for (int k = 0; k < D1; ++k) zero &= pa[(poff[r + 1] - 1) * D1 + k] == 0;
        rep->telescoping_bad += !zero;
    }

    // ---- knots of every hit: k_quantize_hits on records gathered on the device
    DevBuf dinv, dpidx, dps, dpw, dpt, dtc, dla, dkt, dkb, dkc;
    std::vector<int64_t> kt(nh * KN), kb(nh * KN * D1);
    std::vector<int32_t> kc(nh);
    if (nh) {
        std::vector<double> powtau(kMaxDegree, 0.0);
        for (int k = 1; k <= D; ++k) powtau[k - 1] = std::pow(qc.tau, k);
        dinv.ensure(n_ * 4);
        dpidx.ensure(nh * 8);
        dps.ensure(nh * sizeof(sphray_particle));
        dpw.ensure(nh * D * 8);
        dpt.ensure(kMaxDegree * 8);
        dtc.ensure(nh * 8);
        dla.ensure(nh * 8);
        dkt.ensure(kt.size() * 8);
        dkb.ensure(kb.size() * 8);
        dkc.ensure(nh * 4);
        CUDA_OK(cudaMemcpyAsync(dpidx.p, d.hit_pidx.data(), nh * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(dtc.p, d.hit_tchi.data(), nh * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(dla.p, d.hit_lam.data(), nh * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(dpt.p, powtau.data(), kMaxDegree * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemsetAsync(dkt.p, 0, kt.size() * 8, s));
        CUDA_OK(cudaMemsetAsync(dkb.p, 0, kb.size() * 8, s));
        launch_hit_records(d_orig_.as<int32_t>(), n_, dinv.as<int32_t>(), dpidx.as<int64_t>(), nh,
                           d_pxyzh_.as<double4>(), d_mvr_.as<double4>(), d_powh_.as<double>(), D,
                           dps.as<sphray_particle>(), dpw.as<double>(), s);
        QuantParams Q{};
        Q.lut_rows = d_lut_.as<double>();
        Q.lut_stride = lut_.m + lut_.nj;
        Q.lut_N = lut_.N;
        Q.lut_dl = lut_.delta_lambda;
        Q.q = lut_.q;
        Q.K = lut_.K;
        Q.m = lut_.m;
        Q.tau = qc.tau;
        Q.sigma = qc.sigma;
        Q.inv_tau = recip_or_nan(qc.tau);
        Q.inv_dl = recip_or_nan(lut_.delta_lambda);
        Q.w32 = qc.int_width == 32;
        launch_quantize_hits(Q, D, dps.as<sphray_particle>(), dpw.as<double>(), dpt.as<double>(), nh,
                             dtc.as<double>(), dla.as<double>(), dkt.as<int64_t>(), dkb.as<int64_t>(),
                             dkc.as<int32_t>(), s);
        CUDA_OK(cudaMemcpyAsync(kt.data(), dkt.p, kt.size() * 8, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaMemcpyAsync(kb.data(), dkb.p, kb.size() * 8, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaMemcpyAsync(kc.data(), dkc.p, nh * 4, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        for (size_t i = 0; i < nh; ++i)
            if (kc[i] < 0)
                fail(SPHRAY_ERR_OVERFLOW, "validate: quantize overflow", d.hit_pidx[i], d.hit_ray[i]);
    }
    // knots: CSR over the same ray rows as the pieces, sorted by t
    std::vector<std::pair<uint64_t, size_t>> kidx;  // (ray, hit*KN + o)
    for (size_t i = 0; i < nh; ++i)
        for (int o = 0; o < kc[i]; ++o) kidx.emplace_back(d.hit_ray[i], i * KN + o);
    std::sort(kidx.begin(), kidx.end(), [&](const auto& a, const auto& b) {
        return a.first != b.first ? a.first < b.first : kt[a.second] < kt[b.second];
    });
    std::vector<uint64_t> koff(nr + 1, 0);
    std::vector<int64_t> kts(kidx.size()), kbs(kidx.size() * D1);
    {
        size_t r = 0;
        for (size_t i = 0; i < kidx.size(); ++i) {
            while (r < nr && rays[r] < kidx[i].first) koff[++r] = i;
            kts[i] = kt[kidx[i].second];
            for (int k = 0; k < D1; ++k) kbs[i * D1 + k] = kb[kidx[i].second * D1 + k];
        }
        while (r < nr) koff[++r] = kidx.size();
    }

    // group 2: exact superposition (128-bit explicit replay of every piece)
    rep->superposition_rays = nr;
    if (np) {
        DevBuf a, b, c, e, f, g, h, bad;
        a.ensure(koff.size() * 8);
        b.ensure(std::max<size_t>(kts.size(), 1) * 8);
        c.ensure(std::max<size_t>(kbs.size(), 1) * 8);
        e.ensure(poff.size() * 8);
        f.ensure(np * 8);
        g.ensure(np * D1 * 8);
        h.ensure(np * 4);
        bad.ensure(nr * 4);
        CUDA_OK(cudaMemcpyAsync(a.p, koff.data(), koff.size() * 8, cudaMemcpyHostToDevice, s));
        if (!kts.empty()) {
            CUDA_OK(cudaMemcpyAsync(b.p, kts.data(), kts.size() * 8, cudaMemcpyHostToDevice, s));
            CUDA_OK(cudaMemcpyAsync(c.p, kbs.data(), kbs.size() * 8, cudaMemcpyHostToDevice, s));
        }
        CUDA_OK(cudaMemcpyAsync(e.p, poff.data(), poff.size() * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(f.p, pt.data(), np * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(g.p, pa.data(), np * D1 * 8, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemcpyAsync(h.p, prow.data(), np * 4, cudaMemcpyHostToDevice, s));
        CUDA_OK(cudaMemsetAsync(bad.p, 0, nr * 4, s));
        launch_replay(a.as<uint64_t>(), b.as<int64_t>(), c.as<int64_t>(), e.as<uint64_t>(),
                      f.as<int64_t>(), g.as<int64_t>(), h.as<uint32_t>(), np, D, bad.as<unsigned int>(), s);
        std::vector<uint32_t> hb(nr);
        CUDA_OK(cudaMemcpyAsync(hb.data(), bad.p, nr * 4, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        for (size_t r = 0; r < nr; ++r) {
            // the distinct knot positions are exactly the pieces
            size_t distinct = 0;
            for (uint64_t i = koff[r]; i < koff[r + 1]; ++i) distinct += i == koff[r] || kts[i] != kts[i - 1];
            rep->superposition_bad += hb[r] != 0 || distinct != poff[r + 1] - poff[r];
        }
    }

    // group 3: dense-L2 envelope on the first 64 rays (ray-id order)
    {
        const double estar = overall_error(lut_, kCubicKappa);                   // lut.hpp:284-290
        const double qd = quantization_error(lut_, kCubicKappa, kCubicKappaPrime, qc.tau / ds.h_r,
                                             qc.sigma / ds.phi_repr);            // quantize.hpp:64-73
        rep->l2_envelope = 4.0 * std::hypot(estar, qd);
        // h_min over the particles
        std::vector<double4> hx(n_);
        CUDA_OK(cudaMemcpyAsync(hx.data(), d_pxyzh_.p, n_ * sizeof(double4), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        double h_min = n_ ? hx[0].w : 1.0;
        for (size_t i = 0; i < n_; ++i) h_min = std::min(h_min, hx[i].w);
        const double h_step = h_min / 64.0;
        std::vector<uint32_t> ids, rows;
        std::vector<uint64_t> noff{0};
        std::vector<double> t0s, dts;
        std::vector<int> nps;
        for (size_t r = 0; r < nr && ids.size() < 64; ++r) {
            const double t0 = static_cast<double>(pt[poff[r]]) * qc.tau;
            const double t1 = static_cast<double>(pt[poff[r + 1] - 1]) * qc.tau;
            if (!(t1 > t0)) continue;
            int n = std::max(64, static_cast<int>((t1 - t0) / h_step));
            if (n % 2) ++n;  // oracle::simpson (oracle.hpp:38-47)
            ids.push_back(static_cast<uint32_t>(rays[r]));
            rows.push_back(static_cast<uint32_t>(r));
            t0s.push_back(t0);
            dts.push_back((t1 - t0) / n);
            nps.push_back(n);
            noff.push_back(noff.back() + n + 1);
        }
        const size_t nn = noff.back();
        if (!ids.empty()) {
            DevBuf a, b, c, e, f, g, h, ap, ex;
            a.ensure(ids.size() * 4);
            b.ensure(noff.size() * 8);
            c.ensure(ids.size() * 8);
            e.ensure(ids.size() * 8);
            f.ensure(poff.size() * 8);
            g.ensure(rows.size() * 4);
            h.ensure(np * 8 + np * D1 * 8);
            ap.ensure(nn * 8);
            ex.ensure(nn * 8);
            CUDA_OK(cudaMemcpyAsync(a.p, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, s));
            CUDA_OK(cudaMemcpyAsync(b.p, noff.data(), noff.size() * 8, cudaMemcpyHostToDevice, s));
            CUDA_OK(cudaMemcpyAsync(c.p, t0s.data(), t0s.size() * 8, cudaMemcpyHostToDevice, s));
            CUDA_OK(cudaMemcpyAsync(e.p, dts.data(), dts.size() * 8, cudaMemcpyHostToDevice, s));
            CUDA_OK(cudaMemcpyAsync(f.p, poff.data(), poff.size() * 8, cudaMemcpyHostToDevice, s));
            CUDA_OK(cudaMemcpyAsync(g.p, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, s));
            int64_t* dpt_ = h.as<int64_t>();
            CUDA_OK(cudaMemcpyAsync(dpt_, pt.data(), np * 8, cudaMemcpyHostToDevice, s));
            CUDA_OK(cudaMemcpyAsync(dpt_ + np, pa.data(), np * D1 * 8, cudaMemcpyHostToDevice, s));
            const CamConst C = make_camera(cam);
            launch_l2_nodes(C, a.as<uint32_t>(), static_cast<int>(ids.size()), b.as<uint64_t>(),
                            c.as<double>(), e.as<double>(), f.as<uint64_t>(), g.as<uint32_t>(), dpt_,
                            dpt_ + np, D, qc.tau, qc.sigma, d_pxyzh_.as<double4>(), d_mvr_.as<double4>(),
                            n_, ap.as<double>(), ex.as<double>(), s);
            std::vector<double> hap(nn), hex(nn);
            CUDA_OK(cudaMemcpyAsync(hap.data(), ap.p, nn * 8, cudaMemcpyDeviceToHost, s));
            CUDA_OK(cudaMemcpyAsync(hex.data(), ex.p, nn * 8, cudaMemcpyDeviceToHost, s));
            CUDA_OK(cudaStreamSynchronize(s));
            for (size_t r = 0; r < ids.size(); ++r) {
                const int n = nps[r];
                const double hh = dts[r];
                double num = 0.0, den = 0.0;
                for (int i = 0; i <= n; ++i) {
                    const double w = (i == 0 || i == n) ? 1.0 : (i % 2 ? 4.0 : 2.0);
                    const double dv = hap[noff[r] + i] - hex[noff[r] + i];
                    num += w * dv * dv;
                    den += w * hex[noff[r] + i] * hex[noff[r] + i];
                }
                num = std::sqrt(std::max(num * hh / 3.0, 0.0));
                den = std::sqrt(std::max(den * hh / 3.0, 0.0));
                ++rep->l2_rays;
                if (den > 0.0 && num / den > rep->l2_envelope) ++rep->l2_bad;
            }
        }
        rep->l2_fraction_within =
            rep->l2_rays ? static_cast<double>(rep->l2_rays - rep->l2_bad) / rep->l2_rays : 1.0;
    }
    rep->telescoping_pass = rep->telescoping_bad == 0;
    rep->superposition_pass = rep->superposition_bad == 0;
    rep->l2_pass = rep->l2_fraction_within >= 0.95;
    rep->pass = rep->telescoping_pass && rep->superposition_pass && rep->l2_pass;
}

void Engine::render(const sphray_camera& cam, const sphray_tf_point* tf, size_t ntf,
                    const sphray_quanta& qc, const sphray_dataset_stats& ds,
                    const sphray_render_options& opts, double* rgb_host,
                    sphray_render_stats* out, Dumps* dumps) {
    Trace trace;
    set_device();
    const CamConst C = make_camera(cam);  // render_scene: cam.validate() (raycast.hpp:419)
    validate_tf(tf, ntf);                 // raycast.hpp:420
    if (!has_scene_) fail(SPHRAY_ERR_CONFIG, "no scene uploaded");
    if (qc.int_width != 64 && qc.int_width != 32 && qc.int_width != 128)
        fail(SPHRAY_ERR_CONFIG, "int width must be one of 32, 64, 128");
    const bool w32 = qc.int_width == 32, w128 = qc.int_width == 128;
    if (w128) {
        if (dumps)
            fail(SPHRAY_ERR_CONFIG, "int_width 128: the validation outputs hold int64 coefficients");
        // knot positions stay int64 on the device (coefficients and the merge
        // are 128-bit): every position is within |t| < distance to the scene + extent
        const double dx = C.pos[0] - scene_center_[0], dy = C.pos[1] - scene_center_[1],
                     dz = C.pos[2] - scene_center_[2];
        const double reach = std::sqrt(dx * dx + dy * dy + dz * dz) + scene_extent_;
        if (!(reach / qc.tau < 0x1p62))
            fail(SPHRAY_ERR_CAPACITY,
                 "int_width 128: knot positions beyond int64 (t / tau up to " + std::to_string(reach / qc.tau) +
                     ") are not supported on the B200 path");
    }
    const int jb = w128 ? 16 : 8;  // bytes per jump in the window
    const int D = lut_.D, m = lut_.m;
    const double step = opts.step > 0.0 ? opts.step : ds.h_r / 8.0;  // raycast.hpp:424
    const int W = C.W, H = C.H;
    const size_t npix = static_cast<size_t>(W) * H;
    const int tiles_x = (W + kTile - 1) / kTile, tiles_y = (H + kTile - 1) / kTile;
    const uint64_t ntiles = static_cast<uint64_t>(tiles_x) * tiles_y;
    uint64_t owned = (ntiles + nranks_ - 1 - rank_) / nranks_;
    const uint64_t owned_max = (ntiles + nranks_ - 1) / nranks_;
    // pixel region (set_region): the same rays as the full frame, only
    // px in [col_lo, col_hi), py in [row_lo, row_hi)
    int row_lo = 0, row_hi = H, col_lo = 0, col_hi = W, tile_row0 = 0, tile_col0 = 0, tiles_wx = tiles_x;
    if (reg_w_ > 0 && reg_h_ > 0) {
        if (nranks_ > 1) fail(SPHRAY_ERR_CONFIG, "pixel regions need a single-rank context");
        row_lo = std::min(reg_y0_, H);
        row_hi = std::min(reg_y0_ + reg_h_, H);
        col_lo = std::min(reg_x0_, W);
        col_hi = std::min(reg_x0_ + reg_w_, W);
        tile_row0 = row_lo >> kTileShift;
        tile_col0 = col_lo >> kTileShift;
        owned = 0;
        tiles_wx = 0;
        if (row_hi > row_lo && col_hi > col_lo) {
            tiles_wx = ((col_hi - 1) >> kTileShift) - tile_col0 + 1;
            owned = static_cast<uint64_t>(tiles_wx) * (((row_hi - 1) >> kTileShift) - tile_row0 + 1);
        }
    }
    const size_t band_rays = static_cast<size_t>(row_hi - row_lo) * W;  // records / rows copied back
    const int n = static_cast<int>(n_);
    cudaStream_t s = stream_;

    // per-frame uploads: TF (+ per-segment slopes, render_kernel.cuh tf_sample),
    // pow(tau, d) (glibc, quantize.hpp:221)
    h_tf_.assign(ntf * kTfPoint, 0.0);
    for (size_t i = 0; i < ntf; ++i) {
        double* q = &h_tf_[i * kTfPoint];
        q[0] = tf[i].value;
        q[1] = tf[i].r;
        q[2] = tf[i].g;
        q[3] = tf[i].b;
        q[4] = tf[i].absorption;
        if (i + 1 < ntf) {  // d(colour)/d(value) on [value_i, value_i+1]; 0 after the last point
            const double iw = 1.0 / (tf[i + 1].value - tf[i].value);
            q[5] = (tf[i + 1].r - tf[i].r) * iw;
            q[6] = (tf[i + 1].g - tf[i].g) * iw;
            q[7] = (tf[i + 1].b - tf[i].b) * iw;
            q[8] = (tf[i + 1].absorption - tf[i].absorption) * iw;
        }
    }
    d_tf_.ensure(h_tf_.size() * sizeof(double));
    CUDA_OK(cudaMemcpyAsync(d_tf_.p, h_tf_.data(), h_tf_.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    double powtau[kMaxDegree];
    for (int d = 1; d <= D; ++d) powtau[d - 1] = std::pow(qc.tau, d);
    d_powtau_.ensure(sizeof(powtau));
    CUDA_OK(cudaMemcpyAsync(d_powtau_.p, powtau, sizeof(powtau), cudaMemcpyHostToDevice, s));
    d_stats_.ensure(kStatCount * 8);
    CUDA_OK(cudaMemsetAsync(d_stats_.p, 0, kStatCount * 8, s));
    CUDA_OK(cudaMemsetAsync(d_stats_.as<unsigned long long>() + kStatOverflowKey, 0xff, 8, s));
    CUDA_OK(cudaMemsetAsync(d_stats_.as<unsigned long long>() + kStatAccumOverflowRay, 0xff, 8, s));
    d_work_.ensure(16);
    d_retry_count_.ensure(16);
    d_dump_count_.ensure(16);
    CUDA_OK(cudaMemsetAsync(d_dump_count_.p, 0, 16, s));

    CUDA_OK(cudaEventRecord(ev0_, s));
    uint64_t launches = 0;
    // ---- binning (the acceleration structure, hand-written sorts in sort.cu):
    // reference bbox per particle -> depth order of the particles (stable
    // radix sort of the front bounds) -> (tile, particle) entries emitted in
    // depth order -> stable radix sort by tile, so each tile's candidate list
    // is in front order.
    uint64_t entries = 0;
    // rank-local failures are deferred until every rank has reached the
    // collective below (a throw here would leave the other ranks hanging)
    int defer_code = 0;
    std::string defer_msg;
    auto defer = [&](int code, std::string msg) {
        if (!defer_code) {
            defer_code = code;
            defer_msg = std::move(msg);
        }
    };
    d_tile_begin_.ensure(owned_max * 4);
    d_tile_end_.ensure(owned_max * 4);
    CUDA_OK(cudaMemsetAsync(d_tile_begin_.p, 0, owned_max * 4, s));
    CUDA_OK(cudaMemsetAsync(d_tile_end_.p, 0, owned_max * 4, s));
    if (n > 0) {
        const size_t un = static_cast<size_t>(n);
        d_bbox_.ensure(un * sizeof(int4));
        d_front_.ensure(un * sizeof(float));
        d_xy_.ensure(un * 3 * D * sizeof(double));
        d_counts_.ensure(un * 4);
        d_counts2_.ensure(un * 4);
        d_offsets_.ensure(un * 4);
        d_dkeys_.ensure(un * 4);
        d_dkeys2_.ensure(un * 4);
        d_order_.ensure(un * 4);
        d_order2_.ensure(un * 4);
        d_total_.ensure(8);
        d_tmp_.ensure(std::max(radix_tmp_bytes(un), scan_tmp_bytes(un)));
        PrepParams pp{};
        pp.cam = C;
        pp.n = n;
        pp.D = D;
        pp.q = lut_.q;
        pp.reach_scale = std::max(lut_.theta_max, lut_.q);
        pp.pxyzh = d_pxyzh_.as<double4>();
        pp.mvr = d_mvr_.as<double4>();
        pp.powh = d_powh_.as<double>();
        pp.powtau = d_powtau_.as<double>();
        pp.sigma = qc.sigma;
        pp.bbox = d_bbox_.as<int4>();
        pp.front = d_front_.as<float>();
        pp.xy = d_xy_.as<double>();
        pp.counts = d_counts_.as<uint32_t>();
        pp.tiles_x = tiles_x;
        pp.rank = rank_;
        pp.nranks = nranks_;
        launch_prep(pp, s);
        launch_depth_keys(d_front_.as<float>(), n, d_dkeys_.as<uint32_t>(), d_order_.as<uint32_t>(), s);
        const bool o2 = sort_pairs_u32(d_dkeys_.as<uint32_t>(), d_dkeys2_.as<uint32_t>(), d_order_.as<uint32_t>(),
                                       d_order2_.as<uint32_t>(), un, 32, d_tmp_.p, s);
        const uint32_t* order = o2 ? d_order2_.as<uint32_t>() : d_order_.as<uint32_t>();
        CUDA_OK(cudaMemsetAsync(d_total_.p, 0, 8, s));
        launch_gather_counts(d_counts_.as<uint32_t>(), order, n, d_counts2_.as<uint32_t>(),
                             d_total_.as<unsigned long long>(), s);
        scan_u32(d_counts2_.as<uint32_t>(), d_offsets_.as<uint32_t>(), un, d_tmp_.p, nullptr, s);
        unsigned long long total = 0;
        CUDA_OK(cudaMemcpyAsync(&total, d_total_.p, 8, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        launches += 2 + 3 * radix_passes(32) + 1 + 3;  // prep, depth keys, sort, gather, scan
        trace.mark("prep+depth+scan");
        if (total >= 0xffffffffull) {
            defer(SPHRAY_ERR_CAPACITY, "more than 2^32 (tile, particle) entries; shard over more ranks");
        } else {
            entries = total;
        }
        if (entries > 0) {
            d_keys_.ensure(entries * 4);
            d_keys2_.ensure(entries * 4);
            d_vals_.ensure(entries * 4);
            d_vals2_.ensure(entries * 4);
            d_tmp_.ensure(radix_tmp_bytes(entries));
            launch_emit(pp, order, d_offsets_.as<uint32_t>(), d_keys_.as<uint32_t>(), d_vals_.as<uint32_t>(), s);
            const int end_bit = bits_for(owned_max - 1);  // tile keys are < owned_max
            const bool k2 = sort_pairs_u32(d_keys_.as<uint32_t>(), d_keys2_.as<uint32_t>(), d_vals_.as<uint32_t>(),
                                           d_vals2_.as<uint32_t>(), entries, end_bit, d_tmp_.p, s);
            const uint32_t* cand = k2 ? d_vals2_.as<uint32_t>() : d_vals_.as<uint32_t>();
            const uint32_t* tkeys = k2 ? d_keys2_.as<uint32_t>() : d_keys_.as<uint32_t>();
            launch_tile_ranges(tkeys, entries, d_tile_begin_.as<uint32_t>(), d_tile_end_.as<uint32_t>(), s);
            d_cxyzh_.ensure(entries * sizeof(double4));
            d_cmeta_.ensure(entries * sizeof(uint4));
            launch_records(tkeys, cand, entries, d_pxyzh_.as<double4>(), d_bbox_.as<int4>(),
                           d_front_.as<float>(), tiles_x, rank_, nranks_, d_cxyzh_.as<double4>(),
                           d_cmeta_.as<uint4>(), s);
            launches += 1 + 3 * radix_passes(end_bit) + 2;  // emit, sort, ranges, records
        }
    }

    // ---- output buffers
    const bool packed = nranks_ > 1;
    d_image_.ensure(npix * 3 * sizeof(double));
    double* target = d_image_.as<double>();
    if (packed) {
        d_packed_.ensure(owned_max * kTileRays * 3 * sizeof(double));
        CUDA_OK(cudaMemsetAsync(d_packed_.p, 0, owned_max * kTileRays * 3 * sizeof(double), s));
        target = d_packed_.as<double>();
    }

    // ---- render: persistent warps, one ray each at a time
    FrameParams P{};
    P.cam = C;
    P.Q.lut_rows = d_lut_.as<double>();
    P.Q.lut_stride = lut_.m + lut_.nj;
    P.Q.lut_N = lut_.N;
    P.Q.lut_dl = lut_.delta_lambda;
    P.Q.q = lut_.q;
    P.Q.K = lut_.K;
    P.Q.m = lut_.m;
    P.Q.tau = qc.tau;
    P.Q.sigma = qc.sigma;
    P.Q.inv_tau = recip_or_nan(qc.tau);
    P.Q.inv_dl = recip_or_nan(lut_.delta_lambda);
    P.Q.w32 = w32 ? 1 : 0;
    P.n = n;
    P.pxyzh = d_pxyzh_.as<double4>();
    P.xy = d_xy_.as<double>();
    P.bbox = d_bbox_.as<int4>();
    P.front = d_front_.as<float>();
    P.orig = d_orig_.as<int32_t>();
    P.cxyzh = d_cxyzh_.as<double4>();
    P.cmeta = d_cmeta_.as<uint4>();
    P.tile_begin = d_tile_begin_.as<uint32_t>();
    P.tile_end = d_tile_end_.as<uint32_t>();
    P.tiles_x = tiles_x;
    P.tiles_y = tiles_y;
    P.rank = rank_;
    P.nranks = nranks_;
    P.inv_tau = 1.0 / qc.tau;
    P.inv_step = 1.0 / step;
    P.tf = d_tf_.as<double>();
    P.ntf = static_cast<int>(ntf);
    P.tf0_clear = tf_absorption_at_zero(tf, ntf) == 0.0;
    P.step = step;
    P.bg[0] = opts.background[0];
    P.bg[1] = opts.background[1];
    P.bg[2] = opts.background[2];
    P.mode = opts.mode;
    P.work_counter = d_work_.as<unsigned long long>();
    P.total_work = owned * kTileRays;
    P.rgb = target;
    P.packed = packed;
    P.stats = d_stats_.as<unsigned long long>();
    P.tile_row0 = tile_row0;
    P.tile_col0 = tile_col0;
    P.tiles_wx = tiles_wx;
    P.row_lo = row_lo;
    P.row_hi = row_hi;
    P.col_lo = col_lo;
    P.col_hi = col_hi;
    n_records_ = 0;
    if (record_) {
        const size_t nrec = static_cast<size_t>(row_hi - row_lo) * (col_hi - col_lo);
        d_rec_.ensure(std::max<size_t>(nrec, 1) * sizeof(sphray_ray_record));
        CUDA_OK(cudaMemsetAsync(d_rec_.p, 0, nrec * sizeof(sphray_ray_record), s));
        P.ray_rec = d_rec_.as<sphray_ray_record>();
        n_records_ = nrec;
    }
    P.dump_count = d_dump_count_.as<unsigned long long>();
    d_retry_.ensure(npix * 4);
    d_retry2_.ensure(npix * 4);
    P.retry_list = d_retry_.as<uint32_t>();
    P.retry_count = d_retry_count_.as<unsigned int>();
    if (dumps) {
        if (dumps->hits) {
            const size_t c = std::max<size_t>(dumps->cap_hits, 1);
            d_dump_hr_.ensure(c * 8);
            d_dump_hp_.ensure(c * 8);
            d_dump_hl_.ensure(c * 8);
            d_dump_ht_.ensure(c * 8);
            P.dump_cap_hits = dumps->cap_hits;
            P.dump_hit_ray = d_dump_hr_.as<uint64_t>();
            P.dump_hit_pidx = d_dump_hp_.as<int64_t>();
            P.dump_hit_lam = d_dump_hl_.as<double>();
            P.dump_hit_tchi = d_dump_ht_.as<double>();
        }
        if (dumps->pieces) {
            const size_t c = std::max<size_t>(dumps->cap_pieces, 1);
            d_dump_pr_.ensure(c * 8);
            d_dump_pt_.ensure(c * 8);
            d_dump_pa_.ensure(c * (D + 1) * 8);
            P.dump_cap_pieces = dumps->cap_pieces;
            P.dump_piece_ray = d_dump_pr_.as<uint64_t>();
            P.dump_piece_t = d_dump_pt_.as<int64_t>();
            P.dump_piece_a = d_dump_pa_.as<int64_t>();
        }
        P.mode = SPHRAY_MODE_EXACT;
    }
    // Knot window and CTA shape.  Shared memory (the windows) and registers
    // bound the resident warps; the default window is the largest of a few
    // sizes that reaches the best warps/SM (windows below ~384 slots make
    // config-3 rays overflow into the retry pass).
    const size_t tfb_full = ntf * kTfPoint * sizeof(double);
    // Frames whose rays can span more than ~2^31 position quanta (tiny tau,
    // e.g. degree-1 tables) run the robust variant from the start: it moves
    // the 32-bit window-offset base with every flush.  (The hmax sample above
    // is a heuristic; rays that still overflow go to the robust retry pass.)
    // int_width 32 frames run the robust variant too (its quantize and merge
    // carry the Checked<int32_t> range tests, render_kernel.cuh / quantize.cuh)
    // (P.robust: 1 = rebasing only, 2 = with the int32 range tests.)
    const bool robust_frame = scene_extent_ / qc.tau > 2147483648.0 || w32 || w128;
    P.robust = (w32 || w128) ? 2 : robust_frame ? 1 : 0;
    P.w128 = w128 ? 1 : 0;
    const size_t tfb =
        (tfb_full <= 4096 && !dumps && !w32 && !w128 && !std::getenv("SPHRAY_TF_GLOBAL")) ? tfb_full : 0;
    P.tf_smem = static_cast<int>(tfb);
    auto best_shape = [&](int cap_, int& warps_, int& bps_) {
        const size_t wb_ = warp_smem_bytes(D, cap_, m, jb);
        int best_ = 0;
        warps_ = 1;
        bps_ = 0;
        const char* wenv = std::getenv("SPHRAY_WPB");  // diagnostics: force warps per CTA
        const int wforce = wenv ? std::atoi(wenv) : 0;
        for (int wpb : {4, 2, 8, 1, 3, 6}) {
            if (wforce > 0 && wpb != wforce) continue;
            if (wb_ * wpb + tfb > kSmemLimit) continue;
            const int nb = max_blocks_per_sm(D, m, wpb, wb_ * wpb + tfb, lut_.K % 2 == 0);
            if (nb * wpb > best_) {
                best_ = nb * wpb;
                warps_ = wpb;
                bps_ = nb;
            }
        }
        return best_;
    };
    int cap = 0, warps = 1, bps = 0;
    // validation dumps (hits / pieces) are written as rays run, so a ray must
    // not be re-run: dump frames use the widest window from the start
    const long long shape_key[4] = {D * 16 + lut_.K + 1024 * jb, m, static_cast<long long>(tfb),
                                    dumps ? -1 : opts.window};
    if (std::equal(shape_key, shape_key + 4, shape_key_)) {
        cap = shape_val_[0];
        warps = shape_val_[1];
        bps = shape_val_[2];
    } else if (dumps) {
        cap = 65535;
        while (cap > 64 && warp_smem_bytes(D, cap, m, jb) + tfb > kSmemLimit) cap = cap * 15 / 16;
        best_shape(cap, warps, bps);
    } else if (opts.window > 0) {
        cap = std::min(opts.window, 65535);
        if (warp_smem_bytes(D, cap, m, jb) + tfb > kSmemLimit)
            fail(SPHRAY_ERR_CONFIG, "knot window does not fit shared memory");
        best_shape(cap, warps, bps);
    } else {
        int best = -1;
        for (int c : {512, 480, 448, 432, 416, 400, 384}) {
            int w_, b_;
            const int r = best_shape(c, w_, b_);
            if (r > best) {
                best = r;
                cap = c;
                warps = w_;
                bps = b_;
            }
        }
    }
    std::copy(shape_key, shape_key + 4, shape_key_);
    shape_val_[0] = cap;
    shape_val_[1] = warps;
    shape_val_[2] = bps;
    const size_t wb = warp_smem_bytes(D, cap, m, jb);
    if (const char* e = std::getenv("SPHRAY_BPS"))  // diagnostics: fewer CTAs per SM
        bps = std::max(1, std::min(bps, std::atoi(e)));
    if (bps < 1) bps = 1;
    P.cap = cap;
    P.warp_bytes = static_cast<int>(wb);
    if (trace.on)
        trace.line += " cap=" + std::to_string(cap) + " warps/cta=" + std::to_string(warps) +
                      " ctas/sm=" + std::to_string(bps);
    CUDA_OK(cudaMemsetAsync(d_work_.p, 0, 8, s));
    CUDA_OK(cudaMemsetAsync(d_retry_count_.p, 0, 8, s));
    if (reg_w_ > 0 && reg_h_ > 0 && band_rays > 0) {
        // region frames: the rows handed back show the background outside the region
        launch_fill_bg(d_image_.as<double>() + static_cast<size_t>(row_lo) * W * 3, band_rays,
                       opts.background, s);
        ++launches;
    }
    CUDA_OK(cudaEventRecord(evr0_, s));
    if (defer_code) P.total_work = 0;  // this rank failed: only join the collectives
    if (P.total_work > 0) {
        launch_render(P, D, m, sm_count_ * bps, warps, s);
        ++launches;
    }

    // ---- rays whose window overflowed: once more with the widest window
    trace.mark("launch");
    unsigned retry = 0;
    CUDA_OK(cudaMemcpyAsync(&retry, d_retry_count_.p, 4, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    trace.mark("render");
    // diagnostics (ncu captures of the main launch only): skip the retry pass
    if (std::getenv("SPHRAY_PROFILE_NO_RETRY")) retry = 0;
    if (retry > 0 && dumps) {
        defer(SPHRAY_ERR_CAPACITY, std::to_string(retry) + " rays exceed the widest knot window (" +
                                       std::to_string(cap) + " knots)");
        retry = 0;
    }
    int cap2 = 65535;
    while (cap2 > cap && warp_smem_bytes(D, cap2, m, jb) + tfb > kSmemLimit) cap2 = cap2 * 15 / 16;
    if (retry > 0 && cap2 <= cap) {
        defer(SPHRAY_ERR_CAPACITY, "knot window cannot grow");
        retry = 0;
    }
    if (retry > 0) {
        FrameParams P2 = P;
        P2.cap = cap2;
        P2.warp_bytes = static_cast<int>(warp_smem_bytes(D, cap2, m, jb));
        P2.ray_list = d_retry_.as<uint32_t>();
        P2.tf_smem = 0;  // the robust retry variant reads the TF from global memory
        P2.total_work = retry;
        P2.retry_list = d_retry2_.as<uint32_t>();
        P2.retry_count = d_retry_count_.as<unsigned int>() + 1;
        CUDA_OK(cudaMemsetAsync(d_work_.p, 0, 8, s));
        int bps2 = max_blocks_per_sm(D, m, 1, P2.warp_bytes + tfb, lut_.K % 2 == 0);
        if (bps2 < 1) bps2 = 1;
        launch_render(P2, D, m, std::min<int>(retry, sm_count_ * bps2), 1, s);
        ++launches;
        unsigned retry2 = 0;
        CUDA_OK(cudaMemcpyAsync(&retry2, d_retry_count_.as<unsigned int>() + 1, 4,
                                cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        if (retry2 > 0)
            defer(SPHRAY_ERR_CAPACITY, std::to_string(retry2) + " rays exceed the widest knot window (" +
                                           std::to_string(cap2) + " knots)");
    }
    CUDA_OK(cudaEventRecord(evr1_, s));
    // skipped_particles: counted once (rank 0), the particle set is replicated
    if (rank_ == 0 && n > 0) {
        launch_reach(C, n, lut_.q, d_pxyzh_.as<double4>(), d_bbox_.as<int4>(),
                     d_stats_.as<unsigned long long>() + kStatSkipped, s);
        ++launches;
    }

    // ---- agree on rank-local failures, then gather finished tiles over NCCL
    unsigned long long st[kStatCount];
    if (packed && comm_) {
        auto& a = nccl();
        d_status_.ensure(8 * (nranks_ + 1));
        const long long mine = defer_code;
        CUDA_OK(cudaMemcpyAsync(d_status_.p, &mine, 8, cudaMemcpyHostToDevice, s));
        nccl_ok(a.AllGather(d_status_.p, d_status_.as<long long>() + 1, 1, ncclInt64,
                            static_cast<ncclComm_t>(comm_), s),
                "ncclAllGather(status)");
        std::vector<long long> codes(nranks_);
        CUDA_OK(cudaMemcpyAsync(codes.data(), d_status_.as<long long>() + 1, 8 * nranks_,
                                cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
        for (int r = 0; r < nranks_; ++r)
            if (codes[r])
                fail(static_cast<sphray_status>(codes[r]),
                     r == rank_ ? defer_msg : "rank " + std::to_string(r) + " failed (status " +
                                                  std::to_string(codes[r]) + ")");
        const size_t per_rank = owned_max * kTileRays * 3;
        d_gather_.ensure(per_rank * nranks_ * sizeof(double));
        nccl_ok(a.AllGather(d_packed_.p, d_gather_.p, per_rank, ncclDouble,
                            static_cast<ncclComm_t>(comm_), s),
                "ncclAllGather(tiles)");
        launch_unpack(d_gather_.as<double>(), per_rank, nranks_, tiles_x, W, H, d_image_.as<double>(), s);
        d_stats_all_.ensure(kStatCount * 8 * nranks_);
        nccl_ok(a.AllGather(d_stats_.p, d_stats_all_.p, kStatCount, ncclUint64,
                            static_cast<ncclComm_t>(comm_), s),
                "ncclAllGather(stats)");
        std::vector<unsigned long long> all(kStatCount * nranks_);
        CUDA_OK(cudaMemcpyAsync(all.data(), d_stats_all_.p, all.size() * 8, cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaEventRecord(ev1_, s));
        CUDA_OK(cudaStreamSynchronize(s));
        for (int k = 0; k < kStatCount; ++k)
            st[k] = (k == kStatOverflowKey || k == kStatAccumOverflowRay) ? ~0ull : 0ull;
        for (int r = 0; r < nranks_; ++r)
            for (int k = 0; k < kStatCount; ++k) {
                const unsigned long long v = all[r * kStatCount + k];
                if (k == kStatOverflowKey || k == kStatAccumOverflowRay)
                    st[k] = std::min(st[k], v);
                else if (k == kStatMaxPending)
                    st[k] = std::max(st[k], v);
                else
                    st[k] += v;
            }
    } else {
        if (defer_code) fail(static_cast<sphray_status>(defer_code), defer_msg);
        CUDA_OK(cudaMemcpyAsync(st, d_stats_.p, sizeof(st), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaEventRecord(ev1_, s));
        CUDA_OK(cudaStreamSynchronize(s));
    }
    trace.mark("tail");
    if (trace.on && (st[kStatFlushes] | st[kStatBatches])) {
        static const char* names[] = {"flushes", "scanned", "selected", "chunks", "radix_passes",
                                      "batches", "samples", "balanced", "gather", "resid<128",
                                      "resid<192", "resid<256", "resid<320", "resid<384", "resid>=384",
                                      "bits<=8", "bits<=10", "bits<=12", "bits<=14", "bits<=16",
                                      "bits>16"};
        for (int k = kStatFirstK; k < kStatBits0 + 6; ++k)
            trace.line += std::string(" ") + names[k - kStatFirstK] + "=" + std::to_string(st[k]);
    }
    float ms = 0.0f, ms_bin = 0.0f, ms_render = 0.0f;
    CUDA_OK(cudaEventElapsedTime(&ms, ev0_, ev1_));
    CUDA_OK(cudaEventElapsedTime(&ms_bin, ev0_, evr0_));
    CUDA_OK(cudaEventElapsedTime(&ms_render, evr0_, evr1_));

    if (st[kStatOverflowKey] != ~0ull) {
        // quantize_particle's OverflowError names the particle and ray (quantize.hpp:244-249)
        const int64_t pidx = static_cast<int64_t>(st[kStatOverflowKey] >> 32);
        const uint64_t ray = st[kStatOverflowKey] & 0xffffffffull;
        fail(SPHRAY_ERR_OVERFLOW,
             "quantize: integer overflow (particle " + std::to_string(pidx) + ", ray " +
                 std::to_string(ray) + ")",
             pidx, ray);
    }
    if (st[kStatAccumOverflowRay] != ~0ull) {
        // accumulate's OverflowError names the ray (raycast.hpp:285-289); the
        // GPU raises it only for a genuine overflow of a merged coefficient
        // (the reference's int64 path also throws on spurious Delta t^D
        // intermediates, which the exact wrapped merge does not need)
        const uint64_t ray = st[kStatAccumOverflowRay];
        fail(SPHRAY_ERR_OVERFLOW,
             "accumulate: integer overflow (ray " + std::to_string(ray) + ")", -1, ray);
    }
    if (st[kStatRays] > 0 && !(step > 0.0)) fail(SPHRAY_ERR_CONFIG, "composite: step must be positive");

    if (rgb_host) {
        if (packed && !comm_)  // shard without communicator: this rank's packed tiles
            CUDA_OK(cudaMemcpyAsync(rgb_host, d_packed_.p, owned_max * kTileRays * 3 * sizeof(double),
                                    cudaMemcpyDeviceToHost, s));
        else
            CUDA_OK(cudaMemcpyAsync(rgb_host, d_image_.as<double>() + static_cast<size_t>(row_lo) * W * 3,
                                    band_rays * 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
        CUDA_OK(cudaStreamSynchronize(s));
    }
    if (dumps) {
        unsigned long long dc[2];
        CUDA_OK(cudaMemcpy(dc, d_dump_count_.p, 16, cudaMemcpyDeviceToHost));
        dumps->n_hits = dc[0];
        dumps->n_pieces = dc[1];
        if (dumps->hits && dumps->cap_hits) {
            const size_t k = std::min<size_t>(dc[0], dumps->cap_hits);
            dumps->hit_ray.resize(k);
            dumps->hit_pidx.resize(k);
            dumps->hit_lam.resize(k);
            dumps->hit_tchi.resize(k);
            CUDA_OK(cudaMemcpy(dumps->hit_ray.data(), d_dump_hr_.p, k * 8, cudaMemcpyDeviceToHost));
            CUDA_OK(cudaMemcpy(dumps->hit_pidx.data(), d_dump_hp_.p, k * 8, cudaMemcpyDeviceToHost));
            CUDA_OK(cudaMemcpy(dumps->hit_lam.data(), d_dump_hl_.p, k * 8, cudaMemcpyDeviceToHost));
            CUDA_OK(cudaMemcpy(dumps->hit_tchi.data(), d_dump_ht_.p, k * 8, cudaMemcpyDeviceToHost));
        }
        if (dumps->pieces && dumps->cap_pieces) {
            const size_t k = std::min<size_t>(dc[1], dumps->cap_pieces);
            dumps->piece_ray.resize(k);
            dumps->piece_t.resize(k);
            dumps->piece_a.resize(k * (D + 1));
            CUDA_OK(cudaMemcpy(dumps->piece_ray.data(), d_dump_pr_.p, k * 8, cudaMemcpyDeviceToHost));
            CUDA_OK(cudaMemcpy(dumps->piece_t.data(), d_dump_pt_.p, k * 8, cudaMemcpyDeviceToHost));
            CUDA_OK(cudaMemcpy(dumps->piece_a.data(), d_dump_pa_.p, k * (D + 1) * 8, cudaMemcpyDeviceToHost));
        }
    }
    if (out) {
        sphray_render_stats o{};
        o.particles = n_;
        o.skipped_particles = st[kStatSkipped];
        o.knots = st[kStatKnots];
        o.rays_touched = st[kStatRays];
        o.int_ops = st[kStatIntOps];
        o.residual_failures = st[kStatResidual];
        o.step = step;
        o.hits = st[kStatHits];
        o.candidates = entries;
        o.window_retries = retry;
        o.max_window = st[kStatMaxPending];
        o.device_ms = ms;
        o.bin_ms = ms_bin;
        o.render_ms = ms_render;
        o.launches = launches + (packed && comm_ ? 3 : 0);
        o.terminated_rays = st[kStatTerminated];
        *out = o;
    }
}

void Engine::quantize_hits(const sphray_particle* ps, size_t nhits, const double* tchi,
                           const double* lam, const sphray_lut_view& lutv, const sphray_quanta& qc,
                           int64_t* knot_t, int64_t* knot_b, int32_t* knot_count) {
    set_device();
    const LutHost L = make_lut(lutv);
    if (qc.int_width == 128)
        fail(SPHRAY_ERR_CONFIG, "int_width 128: quantize_hits returns int64 jumps");
    if (nhits == 0) return;
    const int D = L.D, KN = L.K + 1;
    std::vector<double> powh(nhits * D);
    particle_powers(ps, nhits, D, powh.data());
    double powtau[kMaxDegree];
    for (int d = 1; d <= D; ++d) powtau[d - 1] = std::pow(qc.tau, d);
    DevBuf lut, dps, dpw, dpt, dtc, dla, dkt, dkb, dkc;
    lut.ensure(L.rows.size() * 8);
    dps.ensure(nhits * sizeof(sphray_particle));
    dpw.ensure(powh.size() * 8);
    dpt.ensure(sizeof(powtau));
    dtc.ensure(nhits * 8);
    dla.ensure(nhits * 8);
    dkt.ensure(nhits * KN * 8);
    dkb.ensure(nhits * KN * (D + 1) * 8);
    dkc.ensure(nhits * 4);
    CUDA_OK(cudaMemcpy(lut.p, L.rows.data(), L.rows.size() * 8, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dps.p, ps, nhits * sizeof(sphray_particle), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dpw.p, powh.data(), powh.size() * 8, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dpt.p, powtau, sizeof(powtau), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dtc.p, tchi, nhits * 8, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(dla.p, lam, nhits * 8, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemset(dkt.p, 0, nhits * KN * 8));
    CUDA_OK(cudaMemset(dkb.p, 0, nhits * KN * (D + 1) * 8));
    QuantParams Q{};
    Q.lut_rows = lut.as<double>();
    Q.lut_stride = L.m + L.nj;
    Q.lut_N = L.N;
    Q.lut_dl = L.delta_lambda;
    Q.q = L.q;
    Q.K = L.K;
    Q.m = L.m;
    Q.tau = qc.tau;
    Q.sigma = qc.sigma;
    Q.inv_tau = recip_or_nan(qc.tau);
    Q.inv_dl = recip_or_nan(L.delta_lambda);
    Q.w32 = qc.int_width == 32;
    launch_quantize_hits(Q, D, dps.as<sphray_particle>(), dpw.as<double>(), dpt.as<double>(), nhits,
                         dtc.as<double>(), dla.as<double>(), dkt.as<int64_t>(), dkb.as<int64_t>(),
                         dkc.as<int32_t>(), stream_);
    CUDA_OK(cudaStreamSynchronize(stream_));
    CUDA_OK(cudaMemcpy(knot_t, dkt.p, nhits * KN * 8, cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(knot_b, dkb.p, nhits * KN * (D + 1) * 8, cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(knot_count, dkc.p, nhits * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < nhits; ++i)
        if (knot_count[i] < 0)
            fail(SPHRAY_ERR_OVERFLOW, "quantize: integer overflow (hit " + std::to_string(i) + ")",
                 static_cast<int64_t>(i), 0);
}

}  // namespace sphray_b200
