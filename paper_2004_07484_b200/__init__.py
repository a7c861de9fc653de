"""B200-native differentiable sphere renderer (Pulsar hot path: forward + backward).

The host types and the reference-facing functions import without a GPU; anything that renders
needs the sm_100a library (csrc/libss_b200.so) and a CUDA device -- there is no fallback.
"""
from .types import (AXIS_ANGLE, ORTHOGRAPHIC, PINHOLE, SIX_D, BackwardBuffer, BlendParams, Camera,
                    CameraGradients, ConfigurationError, ContractViolation, DivergenceError, FeatureImage,
                    FormatError, RenderStats, SceneGradients, SoftSphereError, SphereScene, ValidationError,
                    add_sphere_arrays, axis_angle_to_matrix, axis_angle_vjp, camera_from_vector,
                    camera_to_vector, new_scene, rotation_6d_vjp, rotation_from_6d)
from .api import SoftsphereAdapter, render_backward, render_forward
from .engine import CameraSpec, RenderEngine, default_engine
from .function import Renderer, SphereRender
from .optim import (AdamState, DeviceFit, FitConfig, FitResult, Observation, adam_step, fit, photometric_loss,
                    photometric_loss_device)
from .surgery import prune, prune_device, subdivide, subdivide_device
from .sceneio import (import_point_cloud, load_checkpoint, load_checkpoint_device, load_scene, save_checkpoint,
                      save_checkpoint_device, save_scene, scene_from_bytes, scene_from_bytes_device, scene_to_bytes,
                      scene_to_bytes_device)
from .shade import (DirectionalLight, LinearShader, shade_diffuse, shade_diffuse_backward, shade_identity,
                    shade_identity_backward, shade_linear, shade_linear_backward, view_direction_plane)

__version__ = "0.1.0"
