// Compiled and run by tests/test_gpu_sharded.py on a B200: a batch-sharded train_field driven entirely from a C++ host
// (include/sxen_b200_train.hpp over the C ABI, no Python, no CUDA headers).  The reference's layout -- one worker thread per
// contiguous chunk of the batch, accumulators merged in worker order (src/trainer.cpp:93,101-128) -- with every worker
// driving a GPU replica through a LOCAL communicator (sxen_comm_create_local); on a one-GPU box the ranks share device 0.
//   argv: ranks steps batch [device of rank 0] [device of rank 1] ...
// Checks, printed as "key value" lines for the pytest and enforced here too:
//   * every rank ends with bit-identical tables, MLP parameters and loss curve (the exchange sums in rank order, one rank
//     per slice: the reference's fixed merge order)
//   * against a single-GPU twin that ran the same batches whole: the same set of updated table rows, tables and losses
//     within the fp32-accumulation bar
//   * a rejected coordinate in ONE rank's chunk stops the update on EVERY rank (check_input, src/encoding.cpp:183-194)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>

#include "sxen_b200_train.hpp"

using namespace sxen::b200;

#define EXPECT(cond)                                            \
  do {                                                          \
    if (!(cond)) {                                              \
      std::printf("FAILED line %d: %s\n", __LINE__, #cond);     \
      return 1;                                                 \
    }                                                           \
  } while (0)

struct Model {
  HashEncoder encoder;
  Mlp mlp;
  Model(const EncoderConfig& ec, int device, MlpPrecision precision)
      : encoder(ec, device), mlp(MlpConfig{ec.encoded_width(), 64, 2, 1}, device) {
    encoder.init_tables(42);
    mlp.init_params(sxen_hash_combine(42, 1));
    if (precision != MlpPrecision::exact) check(sxen_mlp_set_precision(mlp.handle(), static_cast<int>(precision)));
  }
};

int main(int argc, char** argv) {
  if (argc < 4) {
    std::printf("usage: ranks steps batch [devices...]\n");
    return 2;
  }
  const int ranks = std::atoi(argv[1]);
  std::vector<int> devices(static_cast<std::size_t>(ranks), 0);
  for (int r = 0; r < ranks && 4 + r < argc; ++r) devices[static_cast<std::size_t>(r)] = std::atoi(argv[4 + r]);
  EncoderConfig ec;
  ec.dim = 3;
  ec.levels = 8;
  ec.table_size = 1u << 14;
  ec.features = 2;
  ec.base_resolution = 8;
  ec.growth = 1.6;
  TrainConfig tc;
  tc.steps = std::atoi(argv[2]);
  tc.batch_size = std::atoi(argv[3]);
  tc.record_every = 1;
  tc.level_chunks = 3;  // 8 levels in ranges of 3, 3, 2
  NoiseFieldSpec spec;
  spec.dim = 3;
  spec.kind = NoiseKind::simplex;
  spec.frequency = 5.0;
  const sxen_noise_spec cspec = spec.c();
  const std::uint64_t seed = tc.seed;
  auto make_sampler = [=](int /*rank*/) -> BatchSampler {  // fit_field's batch stream (src/tasks.cpp:156-166)
    return [=](int step, DeviceSpan<double> coords, DeviceSpan<double> /*aux*/, DeviceSpan<double> targets, void* s) {
      check(sxen_sample_field_batch(&cspec, seed, 1, static_cast<std::uint64_t>(step), targets.size, coords.data, targets.data, s));
    };
  };

  for (MlpPrecision precision : {MlpPrecision::exact, MlpPrecision::tensor_bf16x3}) {
    const char* tag = precision == MlpPrecision::exact ? "exact" : "tc";
    if (precision != MlpPrecision::exact && ec.encoded_width() != 16 && ec.encoded_width() != 32) continue;
    std::vector<std::unique_ptr<Model>> models;
    std::vector<Replica> replicas;
    for (int r = 0; r < ranks; ++r) {
      models.push_back(std::make_unique<Model>(ec, devices[static_cast<std::size_t>(r)], precision));
      replicas.push_back(Replica{&models.back()->encoder, &models.back()->mlp, devices[static_cast<std::size_t>(r)], nullptr});
    }
    const TrainResult sharded = train_field_local(replicas, make_sampler, tc);
    EXPECT(sharded.steps_run == tc.steps && static_cast<int>(sharded.loss_curve.size()) == tc.steps);

    Model twin(ec, devices[0], precision);
    TrainConfig one = tc;
    one.queue_window = 1;
    const TrainResult whole = train_field(twin.encoder, twin.mlp, make_sampler(0), one, devices[0]);

    // (1) every rank holds the same model, bit for bit
    Model fresh(ec, devices[0], precision);
    std::size_t updated_rows = 0, updated_rows_twin = 0, row_set_mismatch = 0;
    double worst = 0.0;
    std::size_t off_exact = 0, off_tc = 0;  // entries further from the twin than the exact head's / the tensor-core head's bar
    for (int l = 0; l < ec.levels; ++l) {
      const std::vector<float> t0 = models[0]->encoder.table(l), tw = twin.encoder.table(l), init = fresh.encoder.table(l);
      for (int r = 1; r < ranks; ++r) EXPECT(models[static_cast<std::size_t>(r)]->encoder.table(l) == t0);
      for (std::size_t row = 0; row < t0.size() / 2; ++row) {
        const bool a = t0[2 * row] != init[2 * row] || t0[2 * row + 1] != init[2 * row + 1];
        const bool b = tw[2 * row] != init[2 * row] || tw[2 * row + 1] != init[2 * row + 1];
        updated_rows += a;
        updated_rows_twin += b;
        row_set_mismatch += a != b;
        for (int f = 0; f < 2; ++f) {
          const double d = std::fabs(static_cast<double>(t0[2 * row + f]) - tw[2 * row + f]);
          worst = std::max(worst, d);
          off_exact += d > 2.01e-5;
          off_tc += d > 4.02e-4;
        }
      }
    }
    const std::vector<float> p0 = models[0]->mlp.parameters();
    for (int r = 1; r < ranks; ++r) EXPECT(models[static_cast<std::size_t>(r)]->mlp.parameters() == p0);
    double worst_loss = 0.0;
    for (std::size_t k = 0; k < sharded.loss_curve.size(); ++k)
      worst_loss = std::max(worst_loss, std::fabs(sharded.loss_curve[k].second - whole.loss_curve[k].second) /
                                            std::fabs(whole.loss_curve[k].second));
    std::printf("%s ranks %d updated_rows %zu twin %zu row_set_mismatch %zu table_max_abs_diff %.3g entries_off_exact_bar %zu "
                "entries_off_tc_bar %zu loss_max_rel_diff %.3g first_loss %.17g last_loss %.17g\n",
                tag, ranks, updated_rows, updated_rows_twin, row_set_mismatch, worst, off_exact, off_tc, worst_loss,
                sharded.loss_curve.front().second, sharded.loss_curve.back().second);
    EXPECT(updated_rows > 0);
    // diagnostics for a comparison that fails: the loss curves side by side and where the tables part
    std::printf("diag-%s losses sharded/twin:", tag);
    for (std::size_t k = 0; k < sharded.loss_curve.size(); ++k)
      std::printf(" %.17g/%.17g", sharded.loss_curve[k].second, whole.loss_curve[k].second);
    std::printf("\ndiag-%s entries off the exact bar per level:", tag);
    for (int l = 0; l < ec.levels; ++l) {
      const std::vector<float> t0 = models[0]->encoder.table(l), tw = twin.encoder.table(l);
      std::size_t off = 0;
      for (std::size_t e = 0; e < t0.size(); ++e) off += std::fabs(static_cast<double>(t0[e]) - tw[e]) > 2.01e-5;
      std::printf(" %zu", off);
    }
    std::printf("\n");
  }

  // (2b) reproducible mode: two sharded runs of the same steps end bit-identical to each other (the exchange sums fixed-point words)
  {
    TrainConfig rc = tc;
    rc.reproducible = true;
    std::vector<float> first_run;
    for (int run = 0; run < 2; ++run) {
      std::vector<std::unique_ptr<Model>> models;
      std::vector<Replica> replicas;
      for (int r = 0; r < ranks; ++r) {
        models.push_back(std::make_unique<Model>(ec, devices[static_cast<std::size_t>(r)], MlpPrecision::exact));
        replicas.push_back(Replica{&models.back()->encoder, &models.back()->mlp, devices[static_cast<std::size_t>(r)], nullptr});
      }
      train_field_local(replicas, make_sampler, rc);
      std::vector<float> all;
      for (int l = 0; l < ec.levels; ++l) {
        const std::vector<float> t0 = models[0]->encoder.table(l);
        for (int r = 1; r < ranks; ++r) EXPECT(models[static_cast<std::size_t>(r)]->encoder.table(l) == t0);
        all.insert(all.end(), t0.begin(), t0.end());
      }
      const std::vector<float> p0 = models[0]->mlp.parameters();
      all.insert(all.end(), p0.begin(), p0.end());
      if (run == 0) first_run = all;
      else EXPECT(all == first_run);
    }
    std::printf("reproducible ok\n");
  }

  // (3) a coordinate outside [0,1] in the LAST rank's chunk only: std::invalid_argument, nothing updated on any rank
  {
    std::vector<std::unique_ptr<Model>> models;
    std::vector<Replica> replicas;
    for (int r = 0; r < ranks; ++r) {
      models.push_back(std::make_unique<Model>(ec, devices[static_cast<std::size_t>(r)], MlpPrecision::exact));
      replicas.push_back(Replica{&models.back()->encoder, &models.back()->mlp, devices[static_cast<std::size_t>(r)], nullptr});
    }
    const std::size_t batch = static_cast<std::size_t>(tc.batch_size);
    auto bad_sampler = [=](int rank) -> BatchSampler {
      const int dev = devices[static_cast<std::size_t>(rank)];
      return [=](int step, DeviceSpan<double> coords, DeviceSpan<double>, DeviceSpan<double> targets, void* s) {
        check(sxen_sample_field_batch(&cspec, seed, 1, static_cast<std::uint64_t>(step), targets.size, coords.data, targets.data, s));
        if (step == 1) {
          const double outside = 1.25;
          check(sxen_device_upload(dev, coords.data + (batch - 1) * 3 + 1, &outside, sizeof(double), s));
        }
      };
    };
    TrainConfig two = tc;
    two.steps = 3;
    bool threw = false;
    std::string what;
    try {
      train_field_local(replicas, bad_sampler, two);
    } catch (const std::invalid_argument& e) {
      threw = true;
      what = e.what();
    }
    EXPECT(threw);
    // step 0 was applied everywhere, step 1 nowhere: all ranks still agree bit for bit
    for (int l = 0; l < ec.levels; ++l)
      for (int r = 1; r < ranks; ++r) EXPECT(models[static_cast<std::size_t>(r)]->encoder.table(l) == models[0]->encoder.table(l));
    std::printf("rejected %s\n", what.c_str());
  }
  std::printf("sharded ok\n");
  return 0;
}
