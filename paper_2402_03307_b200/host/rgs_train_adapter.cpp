// Drop-in C++ implementation of the reference's training-side entry points over the C ABI.
//
// A maintainer compiles this file INSTEAD OF src/image.cpp, src/ssim.cpp, src/loss.cpp,
// src/knn.cpp and src/optim.cpp (next to host/rgs_adapter.cpp, which replaces
// src/rasterizer.cpp) and links librgs_cuda.so.  Every declaration of image.hpp, ssim.hpp,
// loss.hpp, knn.hpp and optim.hpp keeps its signature, argument meaning and exceptions:
//   psnr / l1_loss / l1_loss_backward   image.cpp      -> rgs_image_loss_f64
//   ssim_loss / ssim_loss_with_grad     ssim.cpp       -> rgs_image_loss_f64 (FP64, reference order)
//   entropy_loss(_with_grad)            loss.cpp:16-31 -> rgs_entropy_loss
//   consistency_loss                    loss.cpp:33-58 -> rgs_consistency_loss
//   KdTree4::knn / build_knn4d          knn.cpp        -> rgs_knn_query (exact grid KNN)
//   adam_step / accumulate_stats        optim.cpp      -> rgs_adam_step / rgs_accumulate_stats
//   densify_and_prune / reset_opacity   optim.cpp      -> rgs_densify_and_prune / rgs_reset_opacity
//   initialize_scene                    optim.cpp:53-108 (host draws; nearest neighbours on the device)
// The store is host-resident in the reference's API, so each call stages it through the
// device (an FP64 scene: the doubles reach the kernels unrounded).  A device-resident loop
// should call the C ABI directly.  Differences a caller sees: adam_step
// takes the gradient through float32 (the device gradient format); `threads` is ignored;
// KdTree4::knn supports k <= 16; consistency_loss needs equally long neighbour lists (as
// build_knn4d produces); images must have 3 channels.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "rgs/image.hpp"
#include "rgs/knn.hpp"
#include "rgs/loss.hpp"
#include "rgs/optim.hpp"
#include "rgs/sh.hpp"
#include "rgs/ssim.hpp"
#include "rgs_cuda.h"
#include "rgs_dropin_common.hpp"

namespace rgs {
namespace {

rgs_ctx* tctx() { return dropin::context(); }

[[noreturn]] void raise(int rc) {
    const std::string msg = rgs_ctx_last_error(tctx());
    switch (rc) {
        case RGS_E_ZERO_ROTOR: throw ZeroRotorError();
        case RGS_E_NONFINITE_ROTOR: throw NonFiniteRotorError();
        case RGS_E_DEGENERATE_TIME: throw DegenerateTimeError();
        default: throw std::runtime_error(msg.rfind("ssim:", 0) == 0 ? msg : "rgs_b200: " + msg);
    }
}
void check(int rc) {
    if (rc != RGS_OK) raise(rc);
}

// Device buffer borrowed from the drop-ins' pool for the duration of a call.
struct Dev {
    void* p = nullptr;
    explicit Dev(size_t bytes) { p = dropin::pool_get(bytes); }
    ~Dev() { dropin::pool_put(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
    void put(const void* src, size_t bytes) { check(rgs_memcpy(tctx(), p, src, bytes)); }
    void get(void* dst, size_t bytes) const { check(rgs_memcpy(tctx(), dst, p, bytes)); }
};

// ---------------------------------------------------------------- images
struct ImageLoss {
    double losses[3] = {0, 0, 0};  // l1, ssim, mse
    Image grad;
};

ImageLoss image_loss(const Image& a, const Image& b, double w_l1, double w_ssim, bool want_grad) {
    if (!a.same_shape(b)) throw ShapeMismatchError();
    if (a.channels != 3) throw std::invalid_argument("rgs_b200: images must have 3 channels");
    if (w_ssim != 0 && (a.width < 11 || a.height < 11))
        throw std::runtime_error("ssim: image smaller than the 11x11 window");
    const size_t bytes = a.data.size() * sizeof(double);
    Dev da(bytes), db(bytes), dl(want_grad ? bytes : 8), dloss(3 * sizeof(double));
    da.put(a.data.data(), bytes);
    db.put(b.data.data(), bytes);
    check(rgs_image_loss_f64(tctx(), da.as<double>(), db.as<double>(), a.width, a.height, w_l1, w_ssim, 1.0, 0,
                             want_grad ? dl.as<double>() : nullptr, dloss.as<double>()));
    ImageLoss r;
    dloss.get(r.losses, sizeof r.losses);
    if (want_grad) {
        r.grad = Image(a.width, a.height, a.channels);
        dl.get(r.grad.data.data(), bytes);
    }
    return r;
}

// ---------------------------------------------------------------- store staging
struct DeviceStore {
    rgs_scene* scene = nullptr;
    rgs_optimizer* opt = nullptr;
    ~DeviceStore() {
        if (opt) rgs_optimizer_destroy(opt);
        if (scene) rgs_scene_destroy(scene);
    }
};

// The device copy of the last store an optimizer entry point (adam_step, accumulate_stats,
// reset_opacity) worked on: parameters, moments and statistics, with the hashes of the host
// store it was last synchronised with.  While the host store still hashes to them (train_from
// changes it only through these entry points) the next call skips the upload.
struct Mirror {
    DeviceStore d;
    int n = -1;
    uint64_t hp = 0, hm = 0, hs = 0;
    long long uploads = 0, reuses = 0;
};
Mirror& mirror() {
    static Mirror m;
    return m;
}

void rows65(const GaussianStore& s, bool moments_v, std::vector<double>& out) {
    const size_t n = (size_t)s.size();
    out.resize(65 * n);
    dropin::parallel_for(n, [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) {
            double* r = out.data() + 65 * i;
            const Vec4& mm = moments_v ? s.v_mean[i] : s.m_mean[i];
            const Vec4& ml = moments_v ? s.v_ls[i] : s.m_ls[i];
            const Vec8& mr = moments_v ? s.v_rot[i] : s.m_rot[i];
            const ShCoeffs& msh = moments_v ? s.v_sh[i] : s.m_sh[i];
            for (int a = 0; a < 4; ++a) r[a] = mm[a], r[4 + a] = ml[a];
            for (int a = 0; a < 8; ++a) r[8 + a] = mr[a];
            r[16] = moments_v ? s.v_op[i] : s.m_op[i];
            for (int ch = 0; ch < 3; ++ch)
                for (int k = 0; k < 16; ++k) r[17 + ch * 16 + k] = msh(ch, k);
        }
    });
}

void upload(const GaussianStore& s, DeviceStore& d, bool with_optimizer) {
    const int n = s.size();
    check(rgs_scene_create_ex(tctx(), n, s.active_sh_degree, RGS_SCENE_F64, &d.scene));
    std::vector<double> mean(4 * (size_t)n), ls(4 * (size_t)n), rot(8 * (size_t)n), op((size_t)n), sh(48 * (size_t)n);
    for (int i = 0; i < n; ++i) {
        for (int a = 0; a < 4; ++a) mean[4 * i + a] = s.mean[i][a], ls[4 * i + a] = s.log_scales[i][a];
        const Vec8 c = s.rotor[i].coeffs();
        for (int a = 0; a < 8; ++a) rot[8 * i + a] = c[a];
        op[i] = s.opacity_logit[i];
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) sh[48 * (size_t)i + ch * 16 + k] = s.sh[i](ch, k);
    }
    if (n) check(rgs_scene_upload_f64(tctx(), d.scene, mean.data(), ls.data(), rot.data(), op.data(), sh.data(), nullptr));
    if (!with_optimizer) return;
    check(rgs_optimizer_create(tctx(), d.scene, &d.opt));
    if (!n) return;
    std::vector<double> m, v, acc((size_t)n);
    std::vector<int32_t> cnt((size_t)n);
    rows65(s, false, m);
    rows65(s, true, v);
    for (int i = 0; i < n; ++i) acc[i] = s.grad_accum[i], cnt[i] = s.grad_count[i];
    check(rgs_optimizer_upload(tctx(), d.opt, m.data(), v.data(), acc.data(), cnt.data()));
}

// Device store -> host store (resized to the device size; active_sh_degree kept).
void download(const DeviceStore& d, GaussianStore& s) {
    const int n = rgs_scene_size(d.scene);
    std::vector<double> mean(4 * (size_t)n), ls(4 * (size_t)n), rot(8 * (size_t)n), op((size_t)n), sh(48 * (size_t)n);
    std::vector<double> m(65 * (size_t)n), v(65 * (size_t)n), acc((size_t)n);
    std::vector<int32_t> cnt((size_t)n);
    if (n) {
        check(rgs_scene_download_f64(tctx(), d.scene, mean.data(), ls.data(), rot.data(), op.data(), sh.data()));
        check(rgs_optimizer_download(tctx(), d.opt, m.data(), v.data(), acc.data(), cnt.data()));
    }
    GaussianStore o;
    o.active_sh_degree = s.active_sh_degree;
    for (int i = 0; i < n; ++i) {
        Gaussian4D g;
        for (int a = 0; a < 4; ++a) g.mean[a] = mean[4 * i + a], g.log_scales[a] = ls[4 * i + a];
        Vec8 c;
        for (int a = 0; a < 8; ++a) c[a] = rot[8 * i + a];
        g.rotor = Rotor4::from_coeffs(c);
        g.opacity_logit = op[i];
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) g.sh(ch, k) = sh[48 * (size_t)i + ch * 16 + k];
        o.push_back(g);
        const double* mr = m.data() + 65 * (size_t)i;
        const double* vr = v.data() + 65 * (size_t)i;
        for (int a = 0; a < 4; ++a) {
            o.m_mean[i][a] = mr[a], o.v_mean[i][a] = vr[a];
            o.m_ls[i][a] = mr[4 + a], o.v_ls[i][a] = vr[4 + a];
        }
        for (int a = 0; a < 8; ++a) o.m_rot[i][a] = mr[8 + a], o.v_rot[i][a] = vr[8 + a];
        o.m_op[i] = mr[16];
        o.v_op[i] = vr[16];
        for (int ch = 0; ch < 3; ++ch)
            for (int k = 0; k < 16; ++k) {
                o.m_sh[i](ch, k) = mr[17 + ch * 16 + k];
                o.v_sh[i](ch, k) = vr[17 + ch * 16 + k];
            }
        o.grad_accum[i] = acc[i];
        o.grad_count[i] = cnt[i];
    }
    s = std::move(o);
}

// Parameters / moments of the device store into the host store, in place (sizes equal).
void download_params(const DeviceStore& d, GaussianStore& s) {
    const size_t n = (size_t)s.size();
    double* mean = dropin::scratch<double>(0, 4 * n).data();
    double* ls = dropin::scratch<double>(1, 4 * n).data();
    double* rot = dropin::scratch<double>(2, 8 * n).data();
    double* op = dropin::scratch<double>(3, n).data();
    double* sh = dropin::scratch<double>(4, 48 * n).data();
    check(rgs_scene_download_f64(tctx(), d.scene, mean, ls, rot, op, sh));
    dropin::parallel_for(n, [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) {
            for (int a = 0; a < 4; ++a) s.mean[i][a] = mean[4 * i + a], s.log_scales[i][a] = ls[4 * i + a];
            Vec8 c;
            for (int a = 0; a < 8; ++a) c[a] = rot[8 * i + a];
            s.rotor[i] = Rotor4::from_coeffs(c);
            s.opacity_logit[i] = op[i];
            for (int ch = 0; ch < 3; ++ch)
                for (int k = 0; k < 16; ++k) s.sh[i](ch, k) = sh[48 * i + ch * 16 + k];
        }
    });
}

void download_moments(const DeviceStore& d, GaussianStore& s) {
    const size_t n = (size_t)s.size();
    double* m = dropin::scratch<double>(5, 65 * n).data();
    double* v = dropin::scratch<double>(6, 65 * n).data();
    check(rgs_optimizer_download(tctx(), d.opt, m, v, nullptr, nullptr));
    dropin::parallel_for(n, [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) {
            const double* mr = m + 65 * i;
            const double* vr = v + 65 * i;
            for (int a = 0; a < 4; ++a) {
                s.m_mean[i][a] = mr[a], s.v_mean[i][a] = vr[a];
                s.m_ls[i][a] = mr[4 + a], s.v_ls[i][a] = vr[4 + a];
            }
            for (int a = 0; a < 8; ++a) s.m_rot[i][a] = mr[8 + a], s.v_rot[i][a] = vr[8 + a];
            s.m_op[i] = mr[16];
            s.v_op[i] = vr[16];
            for (int ch = 0; ch < 3; ++ch)
                for (int k = 0; k < 16; ++k) {
                    s.m_sh[i](ch, k) = mr[17 + ch * 16 + k];
                    s.v_sh[i](ch, k) = vr[17 + ch * 16 + k];
                }
        }
    });
}

// The mirror brought in line with the host store: only the parts whose hash changed are
// uploaded (nothing, when the store is the one the last call wrote back).
DeviceStore& synced(const GaussianStore& s) {
    Mirror& m = mirror();
    const int n = s.size();
    const uint64_t hp = dropin::params_hash(s), hm = dropin::moments_hash(s), hs = dropin::stats_hash(s);
    const bool fresh = !m.d.scene || m.n != n;
    if (fresh) {
        m.d.~DeviceStore();
        new (&m.d) DeviceStore();
        m.n = -1;
        check(rgs_scene_create_ex(tctx(), n, s.active_sh_degree, RGS_SCENE_F64, &m.d.scene));
        check(rgs_optimizer_create(tctx(), m.d.scene, &m.d.opt));
    }
    rgs_scene_set_sh_degree(m.d.scene, s.active_sh_degree);
    if (!fresh && m.hp == hp && m.hm == hm && m.hs == hs) {
        ++m.reuses;
        return m.d;
    }
    m.n = -1;  // invalid until every part is up
    if (fresh || m.hp != hp) {
        double* mean = dropin::scratch<double>(0, 4 * (size_t)n).data();
        double* ls = dropin::scratch<double>(1, 4 * (size_t)n).data();
        double* rot = dropin::scratch<double>(2, 8 * (size_t)n).data();
        double* op = dropin::scratch<double>(3, (size_t)n).data();
        double* sh = dropin::scratch<double>(4, 48 * (size_t)n).data();
        dropin::parallel_for((size_t)n, [&](size_t i0, size_t i1) {
            for (size_t i = i0; i < i1; ++i) {
                for (int a = 0; a < 4; ++a) mean[4 * i + a] = s.mean[i][a], ls[4 * i + a] = s.log_scales[i][a];
                const Vec8 c = s.rotor[i].coeffs();
                for (int a = 0; a < 8; ++a) rot[8 * i + a] = c[a];
                op[i] = s.opacity_logit[i];
                for (int ch = 0; ch < 3; ++ch)
                    for (int k = 0; k < 16; ++k) sh[48 * i + ch * 16 + k] = s.sh[i](ch, k);
            }
        });
        if (n) check(rgs_scene_upload_f64(tctx(), m.d.scene, mean, ls, rot, op, sh, nullptr));
    }
    if (n && (fresh || m.hm != hm)) {
        std::vector<double> mo, vo;
        rows65(s, false, mo);
        rows65(s, true, vo);
        check(rgs_optimizer_upload(tctx(), m.d.opt, mo.data(), vo.data(), nullptr, nullptr));
    }
    if (n && (fresh || m.hs != hs)) {
        std::vector<int32_t> cnt((size_t)n);
        for (int i = 0; i < n; ++i) cnt[i] = s.grad_count[i];
        check(rgs_optimizer_upload(tctx(), m.d.opt, nullptr, nullptr, s.grad_accum.data(), cnt.data()));
    }
    m.n = n;
    m.hp = hp;
    m.hm = hm;
    m.hs = hs;
    ++m.uploads;
    return m.d;
}

// After a device update of the mirror written back into `s`: the new hashes, and the new
// parameters published for the render drop-in (a device-to-device copy instead of an upload).
void written_back(const GaussianStore& s, bool params, bool moments, bool stats) {
    Mirror& m = mirror();
    if (params) {
        m.hp = dropin::params_hash(s);
        dropin::publish_params(m.hp, s.size(), s.active_sh_degree, rgs_scene_params_f64(m.d.scene));
    }
    if (moments) m.hm = dropin::moments_hash(s);
    if (stats) m.hs = dropin::stats_hash(s);
}

// Device KNN of `queries` among `points` (exclude[q] skipped), k <= 16.
std::vector<std::vector<int>> knn_device(const std::vector<Vec4>& points, const std::vector<Vec4>& queries,
                                         const std::vector<int32_t>& exclude, int k) {
    if (k > 16) throw std::invalid_argument("rgs_b200: knn supports k <= 16");
    const size_t n = points.size(), nq = queries.size();
    std::vector<double> hp(4 * std::max<size_t>(n, 1)), hq(4 * std::max<size_t>(nq, 1));
    for (size_t i = 0; i < n; ++i)
        for (int a = 0; a < 4; ++a) hp[4 * i + a] = points[i][a];
    for (size_t i = 0; i < nq; ++i)
        for (int a = 0; a < 4; ++a) hq[4 * i + a] = queries[i][a];
    Dev dp(hp.size() * 8), dq(hq.size() * 8), dx(4 * std::max<size_t>(nq, 1)), dout(4 * std::max<size_t>(nq * k, 1));
    dp.put(hp.data(), hp.size() * 8);
    dq.put(hq.data(), hq.size() * 8);
    dx.put(exclude.data(), 4 * nq);
    check(rgs_knn_query(tctx(), dp.as<double>(), (int)n, dq.as<double>(), (int)nq, dx.as<int32_t>(), k,
                        dout.as<int32_t>()));
    std::vector<int32_t> out(nq * (size_t)k);
    if (!out.empty()) dout.get(out.data(), 4 * out.size());
    std::vector<std::vector<int>> r(nq);
    for (size_t q = 0; q < nq; ++q)
        for (int j = 0; j < k; ++j)
            if (out[q * k + j] >= 0) r[q].push_back(out[q * k + j]);
    return r;
}

}  // namespace

// ====================================================================== image.hpp / ssim.hpp
Scalar psnr(const Image& a, const Image& b) {
    const double mse = image_loss(a, b, 1.0, 0.0, false).losses[2];
    if (mse <= 0) return 100;
    return std::min(Scalar(100), 10 * std::log10(1 / mse));
}

Scalar l1_loss(const Image& rendered, const Image& target) {
    return image_loss(rendered, target, 1.0, 0.0, false).losses[0];
}

Image l1_loss_backward(const Image& rendered, const Image& target) {
    return image_loss(rendered, target, 1.0, 0.0, true).grad;
}

Scalar ssim_loss(const Image& rendered, const Image& target) {
    if (!rendered.same_shape(target)) throw ShapeMismatchError();
    if (rendered.width < 11 || rendered.height < 11)
        throw std::runtime_error("ssim: image smaller than the 11x11 window");
    return image_loss(rendered, target, 0.0, 1.0, false).losses[1];
}

Scalar ssim_loss_with_grad(const Image& rendered, const Image& target, Image* grad) {
    if (!rendered.same_shape(target)) throw ShapeMismatchError();
    if (rendered.width < 11 || rendered.height < 11)
        throw std::runtime_error("ssim: image smaller than the 11x11 window");
    ImageLoss r = image_loss(rendered, target, 0.0, 1.0, grad != nullptr);
    if (grad) *grad = std::move(r.grad);
    return r.losses[1];
}

// ====================================================================== loss.hpp
Scalar entropy_loss(const std::vector<Scalar>& opacities) { return entropy_loss_with_grad(opacities, nullptr); }

Scalar entropy_loss_with_grad(const std::vector<Scalar>& opacities, std::vector<Scalar>* grad) {
    if (opacities.empty()) {
        if (grad) grad->clear();
        return 0;
    }
    const size_t n = opacities.size();
    Dev dop(8 * n), dg(8 * n), dl(8);
    dop.put(opacities.data(), 8 * n);
    check(rgs_entropy_loss(tctx(), dop.as<double>(), (int)n, grad ? dg.as<double>() : nullptr, dl.as<double>()));
    double v = 0;
    dl.get(&v, 8);
    if (grad) {
        grad->assign(n, 0.0);
        dg.get(grad->data(), 8 * n);
    }
    return v;
}

Scalar consistency_loss(const std::vector<Vec3>& speeds, const Knn4DIndex& index, std::vector<Vec3>* dL_dspeed) {
    const int n = (int)speeds.size();
    if (n != index.store_size) throw StaleIndexError();
    if (dL_dspeed) dL_dspeed->assign(n, Vec3::Zero());
    if (n == 0) return 0;
    const int k = (int)index.neighbors[0].size();
    std::vector<int32_t> nb((size_t)n * k);
    for (int i = 0; i < n; ++i) {
        if ((int)index.neighbors[i].size() != k)
            throw std::invalid_argument("rgs_b200: consistency_loss needs equally long neighbour lists");
        for (int j = 0; j < k; ++j) nb[(size_t)i * k + j] = index.neighbors[i][j];
    }
    std::vector<double> sp(3 * (size_t)n);
    for (int i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) sp[3 * i + a] = speeds[i][a];
    Dev dsp(8 * sp.size()), dnb(4 * std::max<size_t>(nb.size(), 1)), dg(8 * sp.size()), dl(8);
    dsp.put(sp.data(), 8 * sp.size());
    if (!nb.empty()) dnb.put(nb.data(), 4 * nb.size());
    check(rgs_consistency_loss(tctx(), dsp.as<double>(), n, dnb.as<int32_t>(), k,
                               dL_dspeed ? dg.as<double>() : nullptr, dl.as<double>()));
    double v = 0;
    dl.get(&v, 8);
    if (dL_dspeed) {
        dg.get(sp.data(), 8 * sp.size());
        for (int i = 0; i < n; ++i) (*dL_dspeed)[i] = Vec3(sp[3 * i], sp[3 * i + 1], sp[3 * i + 2]);
    }
    return v;
}

Scalar combine_losses(const LossWeights& w, Scalar l1, Scalar ssim, Scalar entropy, Scalar consistency) {
    return (1 - w.lambda_ssim) * l1 + w.lambda_ssim * ssim + w.lambda_entropy * entropy +
           w.lambda_consistency * consistency;
}

// ====================================================================== knn.hpp
KdTree4::KdTree4(std::vector<Vec4> points) : pts_(std::move(points)) { root_ = pts_.empty() ? -1 : 0; }

std::vector<int> KdTree4::knn(const Vec4& q, int k, int exclude_idx) const {
    if (k <= 0 || pts_.empty()) return {};
    return knn_device(pts_, std::vector<Vec4>{q}, std::vector<int32_t>{exclude_idx}, k)[0];
}

Knn4DIndex build_knn4d(const GaussianStore& store, int k, const Vec4& scene_scales, int) {
    const int n = store.size();
    if (n <= k) throw TooFewPointsError();
    std::vector<Vec4> pts(n);
    for (int i = 0; i < n; ++i) pts[i] = store.mean[i].cwiseQuotient(scene_scales);
    std::vector<int32_t> self(n);
    std::iota(self.begin(), self.end(), 0);
    Knn4DIndex index;
    index.scene_scales = scene_scales;
    index.k = k;
    index.store_size = n;
    index.neighbors = knn_device(pts, pts, self, k);
    return index;
}

// ====================================================================== optim.hpp
void TrainConfig::validate() const {
    auto ok = [](Scalar v) { return std::isfinite(v) && v > 0; };
    for (Scalar lr : {lr_position, lr_position_final, lr_scales, lr_rotor, lr_sh_dc, lr_sh_rest, lr_opacity})
        if (!ok(lr)) throw std::invalid_argument("TrainConfig: learning rates must be positive");
    if (batch < 1 || total_steps < 0) throw std::invalid_argument("TrainConfig: batch must be >= 1");
    if (std::min({densify_interval, opacity_reset_interval, knn_rebuild_interval, sh_unlock_interval}) <= 0)
        throw std::invalid_argument("TrainConfig: intervals must be positive");
    if (init_count < 1) throw std::invalid_argument("TrainConfig: init_count must be >= 1");
    for (int a = 0; a < 3; ++a)
        if (!(box_max[a] > box_min[a])) throw std::invalid_argument("TrainConfig: init box is empty");
    if (min_gaussians < 1 || max_gaussians < min_gaussians)
        throw std::invalid_argument("TrainConfig: bad gaussian count bounds");
    if (!ok(init_time_scale) || !(init_opacity > 0) || !(init_opacity < 1))
        throw std::invalid_argument("TrainConfig: bad initialization constants");
}

Scalar lr_schedule(int step, int total, Scalar lr_init, Scalar lr_final) {
    if (total <= 0) return lr_init;
    const Scalar u = std::clamp((Scalar)step / (Scalar)total, Scalar(0), Scalar(1));
    return lr_init * std::pow(lr_final / lr_init, u);
}

namespace {

// optim.cpp:53-90: scales from the nearest spatial neighbour (device KNN, k = 1).
GaussianStore seed_store(const std::vector<Vec4>& points, const std::vector<Vec3>& colors, const TrainConfig& config) {
    const int n = (int)points.size();
    std::vector<Scalar> nn(n, 0);
    if (n > 1) {
        std::vector<Vec4> spatial(n);
        for (int i = 0; i < n; ++i) spatial[i] = Vec4(points[i][0], points[i][1], points[i][2], 0);
        std::vector<int32_t> self(n);
        std::iota(self.begin(), self.end(), 0);
        const auto nb = knn_device(spatial, spatial, self, 1);
        for (int i = 0; i < n; ++i) nn[i] = (spatial[nb[i][0]] - spatial[i]).norm();
    } else {
        nn[0] = 0.1 * (config.box_max - config.box_min).norm();
    }
    const Scalar st = config.static_mode ? kStaticTemporalScale : config.init_time_scale;
    const Scalar logit = std::log(config.init_opacity / (1 - config.init_opacity));
    GaussianStore store;
    for (int i = 0; i < n; ++i) {
        Gaussian4D g;
        g.mean = points[i];
        const Scalar s = std::max(nn[i], Scalar(1e-7));
        g.log_scales = Vec4(std::log(s), std::log(s), std::log(s), std::log(st));
        g.rotor = Rotor4::identity();
        g.opacity_logit = logit;
        g.sh = ShCoeffs::Zero();
        if (!colors.empty())
            for (int ch = 0; ch < 3; ++ch) g.sh(ch, 0) = (colors[i][ch] - 0.5) / kShC0;
        store.push_back(g);
    }
    return store;
}

}  // namespace

GaussianStore initialize_scene(const TrainConfig& config, std::mt19937_64& rng) {
    config.validate();
    std::uniform_real_distribution<Scalar> uni(0, 1);
    std::vector<Vec4> points(config.init_count);
    for (auto& p : points) {
        for (int a = 0; a < 3; ++a) p[a] = config.box_min[a] + uni(rng) * (config.box_max[a] - config.box_min[a]);
        p[3] = config.static_mode ? Scalar(0.5) : uni(rng);
    }
    return seed_store(points, {}, config);
}

GaussianStore initialize_scene(const std::vector<Vec4>& points, const std::vector<Vec3>& colors,
                               const TrainConfig& config) {
    config.validate();
    if (points.empty()) throw EmptySourceError();
    if (!colors.empty() && colors.size() != points.size())
        throw std::invalid_argument("initialize_scene: colors/points size mismatch");
    return seed_store(points, colors, config);
}

void adam_step(GaussianStore& store, const StoreGrads& grads, const TrainConfig& config, int step) {
    if (grads.size() != store.size()) throw ShapeMismatchGradError();
    const int n = store.size();
    if (n == 0) return;
    DeviceStore& d = synced(store);
    // gradients in the rgs_scene_params SoA layout (float32, the device gradient format)
    const size_t N = (size_t)n;
    float* g = dropin::scratch<float>(0, 65 * N).data();
    dropin::parallel_for(N, [&](size_t i0, size_t i1) {
        for (size_t i = i0; i < i1; ++i) {
            const GaussianParamGrad& gi = grads.g[i];
            for (int a = 0; a < 4; ++a) {
                g[4 * i + a] = (float)gi.d_mean[a];
                g[4 * N + 4 * i + a] = (float)gi.d_log_scales[a];
                g[8 * N + 4 * i + a] = (float)gi.d_rotor[a];
                g[12 * N + 4 * i + a] = (float)gi.d_rotor[4 + a];
            }
            for (int j = 0; j < 48; ++j) {
                const int k = j / 3, ch = j % 3;
                g[(16 + 4 * (size_t)(j / 4)) * N + 4 * i + j % 4] = (float)gi.d_sh(ch, k);
            }
            g[64 * N + i] = (float)gi.d_opacity_logit;
        }
    });
    Dev dg(4 * 65 * N);
    dg.put(g, 4 * 65 * N);
    rgs_adam_config c;
    c.lr_position = config.lr_position;
    c.lr_position_final = config.lr_position_final;
    c.lr_scales = config.lr_scales;
    c.lr_rotor = config.lr_rotor;
    c.lr_sh_dc = config.lr_sh_dc;
    c.lr_sh_rest = config.lr_sh_rest;
    c.lr_opacity = config.lr_opacity;
    c.total_steps = config.total_steps;
    c.static_mode = config.static_mode ? 1 : 0;
    c.lambda_entropy = 0;
    c.accumulate_stats = 0;
    c.flags = 0;
    check(rgs_adam_step(tctx(), d.scene, d.opt, dg.as<float>(), nullptr, nullptr, &c, step, nullptr));
    check(rgs_optimizer_status(tctx(), d.opt));
    download_params(d, store);
    download_moments(d, store);
    written_back(store, true, true, false);
}

void accumulate_stats(GaussianStore& store, const StoreGrads& view_grads) {
    if (view_grads.size() != store.size()) throw ShapeMismatchGradError();
    const int n = store.size();
    if (n == 0) return;
    DeviceStore& d = synced(store);
    std::vector<int32_t> vis(n);
    for (int i = 0; i < n; ++i) vis[i] = view_grads.visible[i];
    Dev dvn(8 * (size_t)n), dvis(4 * (size_t)n);
    dvn.put(view_grads.viewspace_norm.data(), 8 * (size_t)n);
    dvis.put(vis.data(), 4 * (size_t)n);
    check(rgs_accumulate_stats_f64(tctx(), d.opt, dvn.as<double>(), dvis.as<int32_t>()));
    std::vector<int32_t> cnt((size_t)n);
    check(rgs_optimizer_download(tctx(), d.opt, nullptr, nullptr, store.grad_accum.data(), cnt.data()));
    for (int i = 0; i < n; ++i) store.grad_count[i] = cnt[i];
    written_back(store, false, false, true);
}

DensifyReport densify_and_prune(GaussianStore& store, const TrainConfig& config, Scalar scene_extent,
                                std::mt19937_64& rng) {
    DeviceStore d;
    upload(store, d, true);
    // hand the caller's engine to the device call and take it back afterwards
    rgs_rng* r = nullptr;
    check(rgs_rng_create(0, &r));
    std::ostringstream os;
    os << rng;
    check(rgs_rng_set_state(r, os.str().c_str()));
    rgs_densify_config c;
    c.densify_grad_threshold = config.densify_grad_threshold;
    c.percent_dense = config.percent_dense;
    c.split_factor = config.split_factor;
    c.prune_opacity = config.prune_opacity;
    c.min_gaussians = config.min_gaussians;
    c.max_gaussians = config.max_gaussians;
    c.static_mode = config.static_mode ? 1 : 0;
    rgs_densify_report rep{0, 0, 0};
    const int rc = rgs_densify_and_prune(tctx(), d.scene, d.opt, &c, scene_extent, r, &rep);
    size_t len = 0;
    rgs_rng_get_state(r, nullptr, 0, &len);
    std::string st(len, '\0');
    rgs_rng_get_state(r, st.data(), len, &len);
    rgs_rng_destroy(r);
    check(rc);
    std::istringstream is(st);
    is >> rng;
    download(d, store);
    mirror().n = -1;  // the store was resized: the mirror no longer matches it
    DensifyReport out;
    out.cloned = rep.cloned;
    out.split = rep.split;
    out.pruned = rep.pruned;
    return out;
}

void reset_opacity(GaussianStore& store, Scalar value) {
    if (store.size() == 0) return;
    DeviceStore& d = synced(store);
    check(rgs_reset_opacity(tctx(), d.scene, d.opt, value));
    download_params(d, store);
    download_moments(d, store);
    written_back(store, true, true, false);
}

}  // namespace rgs

// Drop-in statistics (bench / tests): optimizer-store uploads and reuses of the device mirror.
extern "C" void rgs_train_adapter_stats(long long* uploads, long long* reuses) {
    if (uploads) *uploads = rgs::mirror().uploads;
    if (reuses) *reuses = rgs::mirror().reuses;
}
