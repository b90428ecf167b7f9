// Example: reference-style C++ call through include/mlsk.hpp (link libmlsk.so).
//   g++ -std=c++17 -Iinclude examples/cpp_reference_api.cpp \
//       -Lpaper_1904_00429_b200/_lib -lmlsk -Wl,-rpath,$PWD/paper_1904_00429_b200/_lib
#include <cstdio>

#include "mlsk.hpp"

using namespace mlsketch_b200;

int main() {
    try {
        // test_estimators.cpp:39-60: constant data collapses every level above zero
        const auto r = mlmc_inner(constant_ones_model(37), target_identity(), LevelPlan{3, 2, {9, 3, 1}}, 77);
        std::printf("value %.1f level1 %.1f\n", r.value, r.per_level[1].estimate);
        // config-2 shapes through the fused DMMA engine
        const auto m = mlmc_matmul(gaussian_mean_matrix_model(256, 4096, 256, 0.5, -1.0, 1.0, 5), target_identity(),
                                   LevelPlan{2, 2, {64, 32, 16}, 32}, 20260823);
        std::printf("config2 value[0] %.6f cost %lld\n", m.value[0], m.total_cost_units);
        // models.cpp:177-227: MC reference value of the deterministic product [[19, 22], [43, 50]]
        const auto ref = reference_matmul(deterministic_matrix_model(), target_identity(), 3, 1);
        std::printf("reference %.1f %.1f %.1f %.1f se %.1f\n", ref.value[0], ref.value[1], ref.value[2],
                    ref.value[3], ref.std_error);
        // two device slots, deterministic virtual shards: the same bits as one device
        EstimatorOptions one, two;
        one.devices = {0};
        one.deterministic = true;
        two.devices = {0, 0};
        two.deterministic = true;
        const auto model = gaussian_mean_matrix_model(128, 4096, 96, 0.5, -1.0, 1.0, 5);
        const LevelPlan small{2, 2, {200, 100, 50}, 32};
        const auto d1 = mlmc_matmul(model, target_identity(), small, 7, one);
        const auto d2 = mlmc_matmul(model, target_identity(), small, 7, two);
        std::printf("deterministic 1 vs 2 devices identical %d\n", d1.value == d2.value ? 1 : 0);
        // session checkpoint / resume: the same bits as an uninterrupted session
        Session a(model, target_identity(), 2, 2, 11, 32);
        a.run_round({70, 33, 10});
        a.run_round({5, 64, 3});
        const auto img = [&] {
            Session b(model, target_identity(), 2, 2, 11, 32);
            b.run_round({70, 33, 10});
            return b.checkpoint();
        }();
        Session c(model, target_identity(), 2, 2, 11, 32);
        c.restore(img);
        c.run_round({5, 64, 3});
        std::printf("resume identical %d\n", a.stats().value == c.stats().value ? 1 : 0);
        return 0;
    } catch (const std::invalid_argument& e) {
        std::printf("invalid_argument: %s\n", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::printf("runtime error: %s\n", e.what());
        return 3;
    }
}
