"""B200-native (sm_100a) TSDF integration — the voxblox (arXiv 1611.03631) hot path.

Product: libvxg.so (hand-written CUDA kernels + C ABI, include/vxg.h) and this
Python mirror of the reference integrator interface (tsdf.py). The CPU oracle
under oracle/ is test infrastructure and is never imported from here.
"""
from .tsdf import (ESDF_VOXEL_DTYPE, DistanceMetric, EsdfConfig, EsdfIntegrator, EsdfLayer, FixedBandMode,
                   QueueMode, K_TSDF_OBSERVED_WEIGHT, VOXEL_DTYPE, MergeMode, Mesh, MeshExtractor, ParseError, Scan, ShardGroup,
                   TimedPose, TsdfConfig, TsdfIntegrator, TsdfLayer, WeightMode, extract_mesh, load_ply_points,
                   load_tum_trajectory, measurement_weight, save_ply_mesh,
                   nccl_unique_id, pose_3x4, projective_distance, raycast, update_tsdf_voxels)

__all__ = ["EsdfConfig", "EsdfIntegrator", "EsdfLayer", "FixedBandMode", "DistanceMetric", "QueueMode",
           "ESDF_VOXEL_DTYPE", "WeightMode", "MergeMode", "TsdfConfig", "Scan", "TsdfLayer", "TsdfIntegrator", "ParseError",
           "ShardGroup", "nccl_unique_id", "Mesh", "MeshExtractor", "extract_mesh",
           "load_ply_points", "load_tum_trajectory", "save_ply_mesh", "TimedPose",
           "projective_distance", "measurement_weight", "update_tsdf_voxels", "raycast", "VOXEL_DTYPE",
           "K_TSDF_OBSERVED_WEIGHT", "pose_3x4"]
