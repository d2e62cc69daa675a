// Runs the GPU parity-task trainer (include/flashrnn/parity.hpp) and prints
// "loss <step> <value>" lines and "final <accuracy>":
//   parity_task <variant 0..3> <dh> <nh> <steps> <batch> <len_max> <warmup> <lr> <seed>
//               <eval_sequences> <eval_len_min> <eval_len_max> <bf16 0|1>
#include <cstdio>
#include <cstdlib>

#include "flashrnn/parity.hpp"

int main(int argc, char** argv) {
  if (argc != 14) return 2;
  namespace T = flashrnn::tasks;
  T::ParityConfig cfg;
  const auto v = static_cast<flashrnn::rnn::Variant>(atoi(argv[1]));
  const int dh = atoi(argv[2]), nh = atoi(argv[3]);
  cfg.steps = atoi(argv[4]);
  cfg.batch_size = atoi(argv[5]);
  cfg.train_len_max = atoi(argv[6]);
  cfg.warmup_steps = atoi(argv[7]);
  const double lr = atof(argv[8]);
  const auto seed = (std::uint64_t)strtoull(argv[9], nullptr, 10);
  cfg.eval_every = 0;
  cfg.eval_sequences = atoi(argv[10]);
  cfg.eval_len_min = atoi(argv[11]);
  cfg.eval_len_max = atoi(argv[12]);
  const T::TrainRun r = atoi(argv[13]) ? T::train_parity_run<flashrnn::rnn::BFloat16>(v, dh, nh, cfg, lr, seed)
                                       : T::train_parity_run<float>(v, dh, nh, cfg, lr, seed);
  for (std::size_t i = 0; i < r.losses.size(); ++i) std::printf("loss %zu %.17g\n", i, r.losses[i]);
  std::printf("final %.17g\n", r.final_accuracy);
  return r.diverged ? 3 : 0;
}
