// drop_in_parity.cpp -- the reference and the B200 build side by side through their C++ APIs
// (fastnn from /root/reference/proj/include, b200nn from include/b200nn.hpp), acceptance-style:
// one PASS/FAIL line per criterion (the gate format of proj/tests/acceptance.cpp:657-685).
// Built by oracle/Makefile into oracle/_ref/drop_in_parity (it links the reference headers);
// run by tests/test_gpu_cpp.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <cstring>
#include <fstream>
#include <iterator>
#include <random>
#include <string>

#include "b200nn.hpp"
#include "fastnn/energy.hpp"
#include "fastnn/network.hpp"

namespace {

double norm_err(const std::vector<float>& got, const fastnn::Tensor& want) {
    double num = 0, den = 0;
    std::size_t i = 0;
    for (std::size_t r = 0; r < want.rows_total(); ++r)
        for (std::size_t j = 0; j < want.last_dim(); ++j, ++i) {
            num = std::max(num, (double)std::fabs(got[i] - want.row_ptr(r)[j]));
            den = std::max(den, (double)std::fabs(want.row_ptr(r)[j]));
        }
    return num / (den > 0 ? den : 1.0);
}

fastnn::Tensor random_batch(std::vector<long long> dims, unsigned seed) {
    fastnn::Tensor t = fastnn::make_tensor(dims);
    std::mt19937 rng(seed);
    std::uniform_real_distribution<float> d(0.0f, 1.0f);
    for (std::size_t r = 0; r < t.rows_total(); ++r)
        for (std::size_t j = 0; j < t.last_dim(); ++j) t.row_ptr(r)[j] = d(rng);
    return t;
}

bool net_criterion(const char* name, const std::vector<long long>& input,
                   const std::vector<fastnn::LayerDesc>& fl, const std::vector<b200nn::LayerDesc>& bl, float lr,
                   std::size_t batch) {
    fastnn::NetworkSpec fs;
    fs.input = input;
    fs.layers = fl;
    fs.lr = lr;
    b200nn::NetworkSpec bs;
    bs.input = input;
    bs.layers = bl;
    bs.lr = lr;
    fastnn::Network ref = fastnn::build_network(fs);
    b200nn::Network dev = b200nn::build_network(bs);
    std::vector<long long> xd{(long long)batch};
    xd.insert(xd.end(), input.begin(), input.end());
    fastnn::Tensor x = random_batch(xd, 1);
    fastnn::Tensor y = fastnn::make_tensor({(long long)batch, 10});
    std::mt19937 lr_rng(2);
    for (std::size_t r = 0; r < batch; ++r) y.at(r, lr_rng() % 10) = 1.0f;
    double worst = 0, dloss = 0;
    for (int step = 0; step < 3; ++step) {
        const double lf = fastnn::train_minibatch(ref, x, y);
        const double lb = b200nn::train_minibatch(dev, x, y);
        dloss = std::max(dloss, std::fabs(lf - lb) / std::fabs(lf));
    }
    auto tp = ref.trainable();
    for (int i = 0; i < dev.num_params(); ++i) worst = std::max(worst, norm_err(dev.param(i), *tp[i].value));
    const bool ok = worst < 1e-3 && dloss < 1e-4;
    std::printf("criterion %s: %s -- 3 steps, loss rel err %.2e, worst param norm err %.2e (tol 1e-3)\n", name,
                ok ? "PASS" : "FAIL", dloss, worst);
    return ok;
}

std::string slurp(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    return std::string((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
}

// fit (network.hpp:488-511) on both sides over the same Dataset, then save_network on both sides
bool fit_checkpoint_criterion() {
    using FL = fastnn::LayerDesc;
    using BL = b200nn::LayerDesc;
    fastnn::NetworkSpec fs;
    fs.input = {1, 28, 28};
    fs.layers = {FL::conv(8, 5, 5), FL::sigmoid(), FL::maxpool(), FL::conv(8, 5, 5), FL::sigmoid(), FL::maxpool(),
                 FL::dense(128, 150), FL::sigmoid(), FL::dense(150, 10), FL::softmax()};
    b200nn::NetworkSpec bs;
    bs.input = fs.input;
    bs.layers = {BL::conv(8, 5, 5), BL::sigmoid(), BL::maxpool(), BL::conv(8, 5, 5), BL::sigmoid(), BL::maxpool(),
                 BL::dense(128, 150), BL::sigmoid(), BL::dense(150, 10), BL::softmax()};
    fastnn::Network ref = fastnn::build_network(fs);
    b200nn::Network dev = b200nn::build_network(bs);
    const std::size_t n = 450;  // 4 full batches of 100 and a partial one
    fastnn::Dataset ds;
    ds.images = random_batch({(long long)n, 1, 28, 28}, 7);
    std::mt19937 lr_rng(8);
    for (std::size_t i = 0; i < n; ++i) ds.labels.push_back((int)(lr_rng() % 10));
    std::vector<float> flat(n * 784);
    for (std::size_t r = 0; r < ds.images.rows_total(); ++r)
        std::memcpy(flat.data() + r * 28, ds.images.row_ptr(r), 28 * sizeof(float));
    const fastnn::TrainReport rf = fastnn::fit(ref, ds, 2);
    const b200nn::TrainReport rd = b200nn::fit(dev, flat.data(), ds.labels.data(), n, 2);
    double dloss = 0, dacc = 0;
    for (int e = 0; e < 2; ++e) {
        dloss = std::max(dloss, std::fabs(rf.epochs[e].loss - rd.epochs[e].loss) / rf.epochs[e].loss);
        dacc = std::max(dacc, std::fabs(rf.epochs[e].accuracy - rd.epochs[e].accuracy));
    }
    double worst = 0;
    auto tp = ref.trainable();
    for (int i = 0; i < dev.num_params(); ++i) worst = std::max(worst, norm_err(dev.param(i), *tp[i].value));
    // the reference's bytes for the device net's parameters: copy them in, save from both sides
    for (int i = 0; i < dev.num_params(); ++i) {
        const std::vector<float> v = dev.param(i);
        std::size_t k = 0;
        for (std::size_t r = 0; r < tp[i].value->rows_total(); ++r)
            for (std::size_t j = 0; j < tp[i].value->last_dim(); ++j) tp[i].value->row_ptr(r)[j] = v[k++];
    }
    fastnn::save_network(ref, "/tmp/b2n_drop_in_ref.fnn1");
    b200nn::save_network(dev, "/tmp/b2n_drop_in_dev.fnn1");
    const bool same = slurp("/tmp/b2n_drop_in_ref.fnn1") == slurp("/tmp/b2n_drop_in_dev.fnn1");
    const bool ok = dloss < 1e-4 && dacc <= 1.0 / n + 1e-12 && worst < 1e-3 && same &&
                    rd.total_batches == rf.total_batches;
    std::printf("criterion fit+checkpoint: %s -- 2 epochs x 450 samples, loss rel err %.2e, accuracy diff %.4f, "
                "worst param norm err %.2e, FNN1 bytes %s\n",
                ok ? "PASS" : "FAIL", dloss, dacc, worst, same ? "identical" : "DIFFER");
    return ok;
}

}  // namespace

// the device generator against std::mt19937 + generate_canonical<double,53>: the state layout the
// header reads (against libstdc++'s own `os << rng`), 10^6 draws bit for bit from a mid-block
// position, the advanced state, and a 5-step cd1_stream whose generator must end where five
// reference cd_k_update calls leave theirs
static bool device_rng_criterion() {
    std::mt19937 g(1234);
    for (int i = 0; i < 77; ++i) g();  // position 77 of the first block
    unsigned st[625];
    b200nn::detail::mt_export(g, st);
    std::ostringstream a, b;
    a << g;
    for (int i = 0; i < 624; ++i) b << st[i] << ' ';
    b << st[624];
    bool ok = a.str() == b.str();
    const long long n = 1000003;
    std::vector<double> dev((size_t)n);
    b200nn::check(b2n_mt19937_draw(0, st, dev.data(), n));
    long long bad = 0;
    for (long long i = 0; i < n; ++i) bad += dev[(size_t)i] != std::generate_canonical<double, 53>(g);
    std::mt19937 back;
    b200nn::detail::mt_import(back, st);
    const bool state_ok = back == g;
    // cd1_stream vs five cd_k_update calls of the reference
    fastnn::Rbm ref(64, 96);
    b200nn::Rbm dev_rbm(64, 96);
    std::mt19937 ia(7), ib(7);
    ref.init(ia);
    dev_rbm.init(ib);
    const std::size_t steps = 5, batch = 20;
    std::vector<float> v(steps * batch * 96);
    std::mt19937 vr(9);
    std::bernoulli_distribution bit(0.3);
    for (float& x : v) x = bit(vr) ? 1.0f : 0.0f;
    std::mt19937 ra(11), rb(11);
    std::vector<double> rr;
    for (std::size_t i = 0; i < steps; ++i) {
        fastnn::Tensor t = fastnn::make_tensor({batch, 96});
        for (std::size_t r = 0; r < batch; ++r)
            for (std::size_t j = 0; j < 96; ++j) t.at(r, j) = v[(i * batch + r) * 96 + j];
        rr.push_back(fastnn::cd_k_update(ref, t, 1, 0.05f, ra));
    }
    const std::vector<double> rd = b200nn::cd1_stream(dev_rbm, v.data(), steps, batch, 0.05f, rb);
    double rec_err = 0.0;
    for (std::size_t i = 0; i < steps; ++i) rec_err = std::max(rec_err, std::fabs(rr[i] - rd[i]) / rr[i]);
    const bool stream_ok = ra == rb && rec_err < 1e-3;
    ok = ok && bad == 0 && state_ok && stream_ok;
    std::printf("criterion device_rng: %s -- layout %s, %lld of %lld draws differ, state %s, cd1_stream rng %s "
                "(recon rel err %.2e)\n",
                ok ? "PASS" : "FAIL", a.str() == b.str() ? "ok" : "DIFFERS", bad, n, state_ok ? "equal" : "DIFFERS",
                ra == rb ? "equal" : "DIFFERS", rec_err);
    return ok;
}

// the op-level layer API: fastnn's conv_forward / conv_backward / pool_forward / pool_backward /
// softmax / softmax_cross_entropy and the b2n_op_* calls on the same fastnn::Tensors, bit for bit
static bool ops_criterion() {
    using b200nn::detail::pack_rows;
    auto same = [](const std::vector<float>& a, const fastnn::Tensor& t) {
        const std::vector<float> b = pack_rows(t);
        return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 4) == 0;
    };
    std::mt19937 g(17);
    std::uniform_real_distribution<float> d(-1.0f, 1.0f);
    auto fill = [&](fastnn::Tensor& t) {
        for (std::size_t r = 0; r < t.rows_total(); ++r)
            for (std::size_t j = 0; j < t.last_dim(); ++j) t.row_ptr(r)[j] = d(g);
    };
    fastnn::ConvShape s;
    s.n = 3, s.c_in = 4, s.k = 6, s.kh = 3, s.kw = 3, s.h = 12, s.w = 10, s.pad = 0;
    fastnn::ConvLayer L(s);
    fill(L.kernels);
    fill(L.b);
    fastnn::Tensor x = fastnn::make_tensor({3, 4, 12, 10});
    fill(x);
    b2n_conv_shape cs{3, 4, 6, 3, 3, 12, 10, 0};
    const fastnn::Tensor y = fastnn::conv_forward(L, x);
    std::vector<float> yb(pack_rows(y).size());
    b200nn::check(b2n_op_conv_forward(0, &cs, pack_rows(x).data(), pack_rows(L.kernels).data(), pack_rows(L.b).data(),
                                      yb.data()));
    bool ok = same(yb, y);
    fastnn::Tensor dy = fastnn::make_tensor({3, 6, 10, 8});
    fill(dy);
    std::vector<float> gk = pack_rows(L.gk), gb = pack_rows(L.gb), dxb(pack_rows(x).size());
    const fastnn::Tensor dx = fastnn::conv_backward(L, x, dy);
    b200nn::check(b2n_op_conv_backward(0, &cs, pack_rows(x).data(), pack_rows(L.kernels).data(), pack_rows(dy).data(),
                                       gk.data(), gb.data(), dxb.data()));
    ok = ok && same(dxb, dx) && same(gk, L.gk) && same(gb, L.gb);
    const fastnn::PoolResult pr = fastnn::pool_forward(fastnn::PoolMode::Max, y);
    std::vector<float> py(pack_rows(pr.y).size()), pa(py.size());
    b200nn::check(b2n_op_pool_forward(0, 0, 3 * 6, 10, 8, yb.data(), py.data(), pa.data()));
    ok = ok && same(py, pr.y) && same(pa, pr.argmax);
    const fastnn::Tensor pdx = fastnn::pool_backward(fastnn::PoolMode::Max, pr.y, pr.argmax);
    std::vector<float> pdxb(pack_rows(pdx).size());
    b200nn::check(b2n_op_pool_backward(0, 0, 3 * 6, 5, 4, py.data(), pa.data(), pdxb.data()));
    ok = ok && same(pdxb, pdx);
    fastnn::Tensor z = fastnn::make_tensor({7, 10});
    fill(z);
    const fastnn::Tensor pz = fastnn::softmax(z);
    std::vector<float> pzb(70);
    b200nn::check(b2n_op_softmax(0, 7, 10, pack_rows(z).data(), pzb.data()));
    fastnn::Tensor lab = fastnn::make_tensor({7, 10});
    for (int r = 0; r < 7; ++r) lab.at(r, (r * 3) % 10) = 1.0f;
    const fastnn::LossGrad lg = fastnn::softmax_cross_entropy(pz, lab);
    std::vector<float> dl(70);
    double loss = 0.0;
    b200nn::check(b2n_op_softmax_cross_entropy(0, 7, 10, pzb.data(), pack_rows(lab).data(), dl.data(), &loss));
    ok = ok && same(pzb, pz) && same(dl, lg.dlogits) && std::fabs(loss - lg.loss) <= 1e-13 * std::fabs(lg.loss);
    std::printf("criterion op_level_api: %s -- conv_forward, conv_backward (dx, gk, gb), pool_forward / backward, "
                "softmax, softmax_cross_entropy bit-identical\n", ok ? "PASS" : "FAIL");
    return ok;
}

int main() {
    using FL = fastnn::LayerDesc;
    using BL = b200nn::LayerDesc;
    bool ok = true;
    ok &= net_criterion("mlp", {784}, {FL::dense(784, 500), FL::sigmoid(), FL::dense(500, 250), FL::sigmoid(),
                                       FL::dense(250, 10), FL::softmax()},
                        {BL::dense(784, 500), BL::sigmoid(), BL::dense(500, 250), BL::sigmoid(), BL::dense(250, 10),
                         BL::softmax()},
                        0.1f, 100);
    ok &= net_criterion("mnist_cnn", {1, 28, 28},
                        {FL::conv(8, 5, 5), FL::sigmoid(), FL::maxpool(), FL::conv(8, 5, 5), FL::sigmoid(),
                         FL::maxpool(), FL::dense(128, 150), FL::sigmoid(), FL::dense(150, 10), FL::softmax()},
                        {BL::conv(8, 5, 5), BL::sigmoid(), BL::maxpool(), BL::conv(8, 5, 5), BL::sigmoid(),
                         BL::maxpool(), BL::dense(128, 150), BL::sigmoid(), BL::dense(150, 10), BL::softmax()},
                        0.1f, 100);
    ok &= net_criterion("cifar_cnn", {3, 32, 32},
                        {FL::conv(12, 5, 5), FL::relu(), FL::maxpool(), FL::conv(12, 5, 5), FL::relu(), FL::maxpool(),
                         FL::dense(300, 64), FL::relu(), FL::dense(64, 10), FL::softmax()},
                        {BL::conv(12, 5, 5), BL::relu(), BL::maxpool(), BL::conv(12, 5, 5), BL::relu(), BL::maxpool(),
                         BL::dense(300, 64), BL::relu(), BL::dense(64, 10), BL::softmax()},
                        0.001f, 100);
    {  // RBM CD-1 with the same generators on both sides
        fastnn::Rbm ref(500, 784);
        b200nn::Rbm dev(500, 784);
        std::mt19937 ia(42), ib(42);
        ref.init(ia);
        dev.init(ib);
        fastnn::Tensor v0 = fastnn::make_tensor({100, 784});
        std::mt19937 vr(3);
        std::bernoulli_distribution bit(0.5);
        for (std::size_t r = 0; r < 100; ++r)
            for (std::size_t j = 0; j < 784; ++j) v0.at(r, j) = bit(vr) ? 1.0f : 0.0f;
        std::mt19937 ra(5), rb(5);
        const double rf = fastnn::cd_k_update(ref, v0, 1, 0.1f, ra);
        const double rd = b200nn::cd_k_update(dev, v0, 1, 0.1f, rb);
        std::vector<float> w, bv, bh;
        dev.get(w, bv, bh);
        const double ew = norm_err(w, ref.w), ev = norm_err(bv, ref.bv), eh = norm_err(bh, ref.bh);
        // the device drew the Bernoulli stream from rb's state: both generators end in the same state
        const bool same_rng = ra == rb;
        const bool r_ok = ew < 1e-3 && ev < 1e-3 && eh < 1e-3 && std::fabs(rf - rd) < 1e-3 * rf && same_rng;
        std::printf("criterion rbm_cd1: %s -- recon %.9g vs %.9g, W %.2e bv %.2e bh %.2e, rng states %s\n",
                    r_ok ? "PASS" : "FAIL", rd, rf, ew, ev, eh, same_rng ? "equal" : "DIFFER");
        ok &= r_ok;
    }
    {  // convolutional RBM CD-1 (crbm_cd_update) with the same generators on both sides
        fastnn::ConvShape s;
        s.c_in = 1;
        s.h = 28;
        s.w = 28;
        s.k = 12;
        s.kh = 5;
        s.kw = 5;
        fastnn::Crbm ref(s);
        b200nn::Crbm dev(1, 28, 28, 12, 5, 5);
        std::mt19937 ia(42), ib(42);
        ref.init(ia);
        dev.init(ib);
        fastnn::Tensor v0 = fastnn::make_tensor({100, 1, 28, 28});
        std::mt19937 vr(3);
        std::bernoulli_distribution bit(0.5);
        for (std::size_t b = 0; b < 100; ++b)
            for (std::size_t y = 0; y < 28; ++y)
                for (std::size_t x = 0; x < 28; ++x) v0.at(b, 0, y, x) = bit(vr) ? 1.0f : 0.0f;
        std::vector<float> k0, bv0, bh0;
        dev.get(k0, bv0, bh0);
        std::mt19937 ra(5), rb(5);
        const double rf = fastnn::crbm_cd_update(ref, v0, 0.1f, ra);
        const double rd = b200nn::crbm_cd_update(dev, v0, 0.1f, rb);
        std::vector<float> kk, bv, bh;
        dev.get(kk, bv, bh);
        const double ek = norm_err(kk, ref.kernels), ev = norm_err(bv, ref.bv), eh = norm_err(bh, ref.bh);
        const bool same_rng = ra == rb;
        const bool c_ok = ek < 1e-3 && ev < 1e-3 && eh < 1e-3 && std::fabs(rf - rd) < 1e-3 * rf && same_rng;
        std::printf("criterion crbm_cd1: %s -- recon %.9g vs %.9g, kernels %.2e bv %.2e bh %.2e, rng states %s\n",
                    c_ok ? "PASS" : "FAIL", rd, rf, ek, ev, eh, same_rng ? "equal" : "DIFFER");
        ok &= c_ok;
    }
    ok &= fit_checkpoint_criterion();
    ok &= device_rng_criterion();
    ok &= ops_criterion();
    return ok ? 0 : 1;
}
