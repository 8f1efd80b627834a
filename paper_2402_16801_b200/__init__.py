"""B200-native batched gridrogue / Craftax environment.

The hot path -- auto-resetting ``env.step`` over thousands of worlds -- runs
as hand-written sm_100a CUDA kernels behind the C ABI of
``include/gridrogue_b200.h`` (``lib/libgridrogue_b200.so``).  Python only
owns the handles and hands torch/numpy buffers to the library.

Public surface (mirrors the reference):
  BatchEnv                       gridrogue_gym.BatchEnv drop-in (numpy I/O)
  GridrogueBatch                 device-resident handle (torch tensors)
  make_craftax_env_from_name     gymnax-style facade (reset(key, params) /
                                 step(key, state, action, params))
  ShardedBatch                   one shard per GPU over torch.distributed
"""

from .env import BatchEnv, GridrogueBatch, TIERS, pixel_shape
from .gymnax import make_craftax_env_from_name, EnvParams, CraftaxEnv, VARIANTS
from .parallel import ShardedBatch, shard_bounds

__all__ = ["BatchEnv", "GridrogueBatch", "TIERS", "pixel_shape", "make_craftax_env_from_name",
           "EnvParams", "CraftaxEnv", "VARIANTS", "ShardedBatch", "shard_bounds"]
__version__ = "0.1.0"
