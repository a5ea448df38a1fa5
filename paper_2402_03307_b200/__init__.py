"""B200-native 4D-rotor Gaussian slicing + splatting (drop-in for the reference renderer path).

The product is librgs_cuda.so (hand-written sm_100a kernels behind include/rgs_cuda.h);
``rgs`` mirrors the reference's renderer API on top of it.
"""
from .rgs import (  # noqa: F401
    Camera,
    CameraError,
    Context,
    DeviceScene,
    GaussianStore,
    MissingRecordsError,
    NonFiniteRotorError,
    RenderOptions,
    RenderOutput,
    RenderRecords,
    RgsUnavailableError,
    StoreGrads,
    ZeroRotorError,
    load_library,
    rasterize_forward,
    render_backward,
    render_flow,
    render_forward,
)
