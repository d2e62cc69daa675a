// Loads an RTN1 file with include/flashrnn/tensor_io.hpp, writes it back, and
// round-trips the parameter bundle: argv[1] in, argv[2] out.
#include <cstdio>

#include "flashrnn/tensor_io.hpp"

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  namespace rnn = flashrnn::rnn;
  const rnn::TensorMap t = rnn::load_tensors(argv[1]);
  rnn::save_tensors(argv[2], t);
  const rnn::Params<double> p = rnn::params_from_tensors(t);
  const rnn::TensorMap back = rnn::params_to_tensors(p);
  if (back.at("recurrent").data != t.at("recurrent").data || back.at("bias").data != t.at("bias").data) return 3;
  try {
    rnn::load_tensors(std::string(argv[1]) + ".missing");
    return 4;
  } catch (const std::invalid_argument&) {
  }
  std::printf("%zu tensors, heads %d gates %d dh %d\n", t.size(), p.num_heads, p.num_gates, p.head_dim);
  return 0;
}
